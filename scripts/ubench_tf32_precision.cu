// Precision probe: how exact is tcgen05.mma.kind::tf32 accumulation over long
// K chains?  One CTA computes D[128 x N] = A[128 x K] B[N x K]^T with
//   mode 1: one pass (operands rounded to tf32 by the MMA)
//   mode 3: 3xTF32 (hi*hi + hi*lo + lo*hi, hi = rna_tf32(x), lo = x - hi)
//   mode 2: 2xFP16 on kind::f16 (hi*hi + hi*lo + lo*hi, hi = f16(x*2^s),
//           lo = f16(x*2^s - hi); per-operand power-of-two scale, undone in
//           the fp32 promotion)
// accumulating in TMEM either over the whole K, or over chunks of KC and then
// added into fp32 registers on the CUDA cores ("promotion").  Errors are
// reported relative to sum_k |a_k b_k| and to max |D| against an fp64 host
// reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tf32p scripts/ubench_tf32_precision.cu
//   /tmp/tf32p
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

constexpr int M = 128, N = 128, KB = 32;   // K block = one 128-B swizzle atom of tf32

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// element (r, k) of a [rows x 64] K-major f16 tile with the 128-B swizzle
__device__ __forceinline__ int swz16(int r, int k) { return r * 64 + ((((k >> 3) ^ (r & 7)) << 3) | (k & 7)); }
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// element (r, k) of a [rows x 32] K-major tile with the 128-B swizzle
__device__ __forceinline__ int swz(int r, int k) { return r * 32 + ((((k >> 2) ^ (r & 7)) << 2) | (k & 3)); }

__global__ void __launch_bounds__(128, 1) k_probe(const float* A, const float* B, int K, int passes, int KC,
                                                  float* D, float sa_s, float sb_s) {
  extern __shared__ uint8_t smem_raw[];
  float* base = (float*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sa[2] = {base, base + M * KB};            // hi, lo
  float* sb[2] = {base + 2 * M * KB, base + 2 * M * KB + N * KB};
  const bool h16 = passes == 2;
  const int kb = h16 ? 2 * KB : KB;   // K elements per 128-B atom row
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  float acc[N];   // thread = row (lane of TMEM), promoted sums
  for (int j = 0; j < N; ++j) acc[j] = 0.f;
  uint32_t phase = 0;
  const uint32_t idesc = h16 ? idesc_f16(M, N) : idesc_tf32(M, N);
  for (int k0 = 0; k0 < K; k0 += kb) {
    if (h16) {
      __half* ha[2] = {(__half*)sa[0], (__half*)sa[1]};
      __half* hb[2] = {(__half*)sb[0], (__half*)sb[1]};
      for (int i = tid; i < M * kb; i += 128) {
        const int r = i / kb, k = i % kb;
        const float v = A[(size_t)r * K + k0 + k] * sa_s;
        const __half h = __float2half_rn(v);
        ha[0][swz16(r, k)] = h;
        ha[1][swz16(r, k)] = __float2half_rn(v - __half2float(h));
      }
      for (int i = tid; i < N * kb; i += 128) {
        const int r = i / kb, k = i % kb;
        const float v = B[(size_t)r * K + k0 + k] * sb_s;
        const __half h = __float2half_rn(v);
        hb[0][swz16(r, k)] = h;
        hb[1][swz16(r, k)] = __float2half_rn(v - __half2float(h));
      }
    } else {
    for (int i = tid; i < M * KB; i += 128) {
      const int r = i / KB, k = i % KB;
      const float v = A[(size_t)r * K + k0 + k];
      const float h = passes == 3 ? tf32_rna(v) : v;
      sa[0][swz(r, k)] = h;
      sa[1][swz(r, k)] = v - h;
    }
    for (int i = tid; i < N * KB; i += 128) {
      const int r = i / KB, k = i % KB;
      const float v = B[(size_t)r * K + k0 + k];
      const float h = passes == 3 ? tf32_rna(v) : v;
      sb[0][swz(r, k)] = h;
      sb[1][swz(r, k)] = v - h;
    }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const bool first_of_chunk = (k0 % KC) == 0;
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kk = 0; kk < KB / 8; ++kk) {
        const uint64_t o = (uint64_t)(kk * 2);   // 32 B per k8 step, in 16-B units
        const int np = passes == 1 ? 1 : 3;
        for (int p = 0; p < np; ++p) {
          const int ia = (p == 2) ? 1 : 0, ib = (p == 1) ? 1 : 0;   // hh, hl, lh
          const uint64_t ad = sdesc_sw128(su32(sa[ia])) + o, bd = sdesc_sw128(su32(sb[ib])) + o;
          const uint32_t accum = (first_of_chunk && kk == 0 && p == 0) ? 0u : 1u;
          if (h16)
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n}" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(accum) : "memory");
          else
            asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n}" ::"r"(tmem),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(accum) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(su32(&bar)), "r"(phase) : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool last_of_chunk = ((k0 + kb) % KC) == 0 || k0 + kb >= K;
    if (last_of_chunk) {
      // drain the chunk's TMEM sum into registers (lane = row = tid)
      for (int j0 = 0; j0 < N; j0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int q = 0; q < 8; ++q) acc[j0 + q] += __uint_as_float(v[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
  }
  const float unscale = 1.f / (sa_s * sb_s);
  for (int j = 0; j < N; ++j) D[(size_t)tid * N + j] = acc[j] * unscale;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

int main() {
  std::mt19937_64 rng(7);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::uniform_real_distribution<float> ud(0.f, 1.f);
  for (int dist : {0, 1})
  for (int K : {256, 1024, 4096}) {
    std::vector<float> A((size_t)M * K), B((size_t)N * K);
    // dist 0: normal; dist 1: relu-like A (half zeros) with magnitudes spread
    // log-uniformly over 2^-20..2^4, B normal scaled by 1e-4 (a gradient)
    for (auto& v : A) v = dist == 0 ? nd(rng) : (ud(rng) < 0.5f ? 0.f : std::exp2(-20.f + 24.f * ud(rng)));
    for (auto& v : B) v = nd(rng) / std::sqrt((float)K) * (dist == 0 ? 1.f : 1e-4f);
    float amax = 0, bmax = 0;
    for (auto v : A) amax = std::max(amax, std::fabs(v));
    for (auto v : B) bmax = std::max(bmax, std::fabs(v));
    std::vector<double> ref((size_t)M * N), mag((size_t)M * N);
    double dmax = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0, m = 0;
        for (int k = 0; k < K; ++k) {
          s += (double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
          m += std::fabs((double)A[(size_t)i * K + k] * B[(size_t)j * K + k]);
        }
        ref[(size_t)i * N + j] = s;
        mag[(size_t)i * N + j] = m;
        dmax = std::max(dmax, std::fabs(s));
      }
    // fp32 sequential FMA reference error (what an FFMA kernel gets)
    double ffma_err = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        float s = 0;
        for (int k = 0; k < K; ++k) s = std::fmaf(A[(size_t)i * K + k], B[(size_t)j * K + k], s);
        ffma_err = std::max(ffma_err, std::fabs(s - ref[(size_t)i * N + j]) / dmax);
      }
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, (size_t)M * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    printf("dist %d K=%d  fp32 FFMA chain: max err %.2e of max|D|\n", dist, K, ffma_err);
    for (int passes : {1, 3, 2})
      for (int headroom : {4, 12})
      for (int KC : {K, 1024, 256, 128, 64}) {
        if (KC > K || (passes != 2 && headroom != 4)) continue;
        // 2xFP16: scale so max|x| * s ~ 2^(15 - headroom)
        const float sa_s = passes == 2 ? std::exp2(std::floor(15 - headroom - std::log2(amax))) : 1.f;
        const float sb_s = passes == 2 ? std::exp2(std::floor(15 - headroom - std::log2(bmax))) : 1.f;
        const int smem = (2 * M * KB + 2 * N * KB) * 4 + 1024;
        CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_probe<<<1, 128, smem>>>(dA, dB, K, passes, KC, dD, sa_s, sb_s);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<float> D((size_t)M * N);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double e_max = 0, e_mag = 0;
        for (size_t t = 0; t < D.size(); ++t) {
          const double e = std::fabs(D[t] - ref[t]);
          e_max = std::max(e_max, e / dmax);
          e_mag = std::max(e_mag, e / mag[t]);
        }
        printf("  passes %d headroom %2d chunk %5d: max err %.2e of max|D|, %.2e of sum|ab|\n", passes, headroom, KC, e_max, e_mag);
      }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  return 0;
}
