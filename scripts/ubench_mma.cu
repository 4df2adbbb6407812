// Micro-benchmark: tcgen05.mma.cta_group::1.kind::tf32 issue rate from one
// smem stage (no TMA), to separate per-instruction overhead from operand
// bandwidth.  Variants: N = 128 / 256, one accumulator (dependent chain) or
// two / three accumulators round-robin.  One CTA per SM, one elected issuer.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_mma scripts/ubench_mma.cu
//   /tmp/ubench_mma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint64_t ad = sdesc_sw128(su32(smem));
    const uint64_t bd = sdesc_sw128(su32(smem + 128 * 128));
    constexpr uint32_t idesc = idesc_tf32(128, N);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tmem + (uint32_t)(((i * 4 + kk) % NACC) * N);
        const uint64_t o = (uint64_t)(kk * 2);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
            "l"(ad + o), "l"(bd + o), "r"(idesc), "r"(1)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar))
        : "memory");
    const long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// cta_group::2: the pair computes a 256 x N tile; CTA r holds A rows [128r, +128)
// and B rows [r N/2, +N/2); the leader issues.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_mma_pair(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (128 + N / 2) * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t ad = sdesc_sw128(su32(smem));
    const uint64_t bd = sdesc_sw128(su32(smem + 128 * 128));
    constexpr uint32_t idesc = idesc_tf32(256, N);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t o = (uint64_t)(kk * 2);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(ad + o), "l"(bd + o), "r"(idesc), "r"(1)
            : "memory");
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(su32(&bar)), "h"((uint16_t)3)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar))
        : "memory");
    const long long t1 = clock64();
    cycles[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
  } else if (threadIdx.x == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int N>
void run_pair(int sms) {
  const int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = (128 + N / 2) * 128 + 2048;
  cudaFuncSetAttribute(k_mma_pair<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma_pair<N><<<sms, 128, smem>>>(iters, d);
  k_mma_pair<N><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms / 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms / 2; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 4.0 * iters;
  const double ideal = mmas * (128.0 * N * 8 * 2) / 4096.0;  // per SM: 128 rows of the pair tile
  printf("pair M=256 N=%d  %s  cycles/mma %.1f  (ideal %.1f)  tensor %.1f%%\n", N,
         cudaGetErrorString(e), mx / mmas, ideal / mmas, 100.0 * ideal / mx);
  cudaFree(d);
}

template <int N, int NACC>
void run(int sms) {
  const int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = (128 + N) * 128 + 2048;
  cudaFuncSetAttribute(k_mma<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma<N, NACC><<<sms, 128, smem>>>(iters, d);
  k_mma<N, NACC><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 4.0 * iters;
  const double ideal = mmas * (128.0 * N * 8 * 2) / 4096.0;  // tf32: 4096 flop/clk/SM
  printf("N=%d acc=%d  %s  cycles/mma %.1f  (ideal %.1f)  tensor %.1f%%\n", N, NACC,
         cudaGetErrorString(e), mx / mmas, ideal / mmas, 100.0 * ideal / mx);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, 1>(sms);
  run<128, 2>(sms);
  run<128, 3>(sms);
  run<256, 1>(sms);
  run<256, 2>(sms);
  run<64, 1>(sms);
  run<64, 4>(sms);
  run_pair<128>(sms);
  run_pair<256>(sms);
  run_pair<64>(sms);
  return 0;
}
