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


// Background TMA-like traffic: one thread keeps 4 x 16 KB cp.async.bulk
// global->smem copies in flight until *done is set; returns bytes copied.
__device__ unsigned long long stream_copies(uint8_t* ring, uint64_t* bars, const uint8_t* src,
                                            volatile int* done) {
  unsigned long long bytes = 0;
  uint32_t phase[4] = {0, 0, 0, 0};
  auto issue = [&](int s, int k) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])),
                 "r"(16384) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(ring + s * 16384)),
        "l"(src + (size_t)(k & 63) * 16384), "r"(16384), "r"(su32(&bars[s]))
        : "memory");
  };
  for (int s = 0; s < 4; ++s) issue(s, s);
  int k = 4;
  while (true) {
    for (int s = 0; s < 4; ++s) {
      asm volatile(
          "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(
              su32(&bars[s])), "r"(phase[s])
          : "memory");
      phase[s] ^= 1;
      bytes += 16384;
      if (*done) return bytes;
      issue(s, k++);
    }
  }
}

template <int N, int NACC, bool BULK = false, int TLD = 0, int SEG = 0>
__global__ void __launch_bounds__(384, 1) k_mma(int iters, unsigned long long* cycles,
                                                const uint8_t* src = nullptr,
                                                unsigned long long* copied = nullptr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint64_t cbars[4];
  __shared__ volatile int done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    done = 0;
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbars[s])));
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
      if (SEG) {
        // dW-like: a "stage" = 4 k8 x 3 MMAs then a commit; a "segment" =
        // SEG stages into one of two accumulators, first MMA overwrites
        const int st = i / 3;
        const uint32_t d = tmem + (uint32_t)(((st / SEG) & 1) * N);
        const int kk = i % 3;
        const uint64_t o = (uint64_t)(kk * 2);
        const uint32_t accum = (st % SEG == 0 && kk == 0) ? 0u : 1u;
        for (int r = 0; r < 4; ++r)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
              "l"(ad + o), "l"(bd + o), "r"(idesc), "r"(r == 0 ? accum : 1u)
              : "memory");
        if (kk == 2) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&cbars[0]))
                       : "memory");
          if (st % SEG == SEG - 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             su32(&cbars[1]))
                         : "memory");
        }
        continue;
      }
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
    done = 1;
  } else if (BULK && threadIdx.x == 32) {
    copied[blockIdx.x] = stream_copies(smem + (128 + N) * 128, cbars, src, &done);
  } else if (TLD && warp >= 4) {
    // epilogue-like TMEM reads of columns [256, 512) (32x32b.x16), TLD = 1:
    // continuous; TLD = n > 1: one 128-column sweep every n * 64 cycles
    const uint32_t q = (uint32_t)(warp & 3) * 32;
    float acc = 0.f;
    unsigned long long reads = 0;
    while (!done) {
      const long long t0 = clock64();
      for (int c = 0; c < 128; c += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
            "%12, %13, %14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15])
            : "r"(tmem + (q << 16) + 256 + (uint32_t)c + (warp >= 8 ? 128u : 0u)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      }
      reads += 128 * 32 * 4;
      if (TLD > 1)
        while (clock64() - t0 < (long long)TLD * 64 && !done) {}
    }
    if (acc == 12345.f) cycles[0] = 0;
    if (copied && (threadIdx.x & 31) == 0) atomicAdd(&copied[blockIdx.x], reads);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// cta_group::2: the pair computes a 256 x N tile; CTA r holds A rows [128r, +128)
// and B rows [r N/2, +N/2); the leader issues.
template <int N, bool BULK = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_mma_pair(int iters, unsigned long long* cycles, const uint8_t* src = nullptr,
               unsigned long long* copied = nullptr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint64_t cbars[4];
  __shared__ volatile int done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < (128 + N / 2) * 32; i += blockDim.x) ((float*)smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    done = 0;
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbars[s])));
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
    done = 1;
  } else if (threadIdx.x == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar))
        : "memory");
    done = 1;
  } else if (BULK && threadIdx.x == 32) {
    copied[blockIdx.x] = stream_copies(smem + (128 + N / 2) * 128, cbars, src, &done);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int N, bool BULK = false>
void run_pair(int sms) {
  const int iters = 4096;
  unsigned long long *d, *cp;
  uint8_t* src;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  cudaMalloc(&cp, sms * sizeof(unsigned long long));
  cudaMalloc(&src, 64 << 14);
  const int smem = (128 + N / 2) * 128 + 2048 + 65536;
  cudaFuncSetAttribute(k_mma_pair<N, BULK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma_pair<N, BULK><<<sms, 128, smem>>>(iters, d, src, cp);
  k_mma_pair<N, BULK><<<sms, 128, smem>>>(iters, d, src, cp);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms / 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms / 2; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 4.0 * iters;
  const double ideal = mmas * (128.0 * N * 8 * 2) / 4096.0;  // per SM: 128 rows of the pair tile
  unsigned long long hc[256];
  cudaMemcpy(hc, cp, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  printf("pair M=256 N=%d bulk=%d  %s  cycles/mma %.1f  (ideal %.1f)  tensor %.1f%%  copy %.1f B/clk\n",
         N, (int)BULK, cudaGetErrorString(e), mx / mmas, ideal / mmas, 100.0 * ideal / mx,
         BULK ? (double)hc[0] / mx : 0.0);
  cudaFree(d);
  cudaFree(cp);
  cudaFree(src);
}

template <int N, int NACC, bool BULK = false, int TLD = 0, int SEG = 0>
void run(int sms) {
  const int iters = 4096;
  unsigned long long *d, *cp;
  uint8_t* src;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  cudaMalloc(&cp, sms * sizeof(unsigned long long));
  cudaMalloc(&src, 64 << 14);
  const int smem = (128 + N) * 128 + 2048 + 65536;
  cudaFuncSetAttribute(k_mma<N, NACC, BULK, TLD, SEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int threads = TLD ? 128 + 256 : 128;
  cudaMemset(cp, 0, sms * sizeof(unsigned long long));
  k_mma<N, NACC, BULK, TLD, SEG><<<sms, threads, smem>>>(iters, d, src, cp);
  cudaMemset(cp, 0, sms * sizeof(unsigned long long));
  k_mma<N, NACC, BULK, TLD, SEG><<<sms, threads, smem>>>(iters, d, src, cp);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 4.0 * iters;
  const double ideal = mmas * (128.0 * N * 8 * 2) / 4096.0;  // tf32: 4096 flop/clk/SM
  unsigned long long hc[256];
  cudaMemcpy(hc, cp, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  printf("seg=%d N=%d acc=%d bulk=%d tld=%d  %s  cycles/mma %.1f  (ideal %.1f)  tensor %.1f%%  copy/tmem-read %.1f B/clk\n",
         SEG, N, NACC, (int)BULK, TLD, cudaGetErrorString(e), mx / mmas, ideal / mmas, 100.0 * ideal / mx,
         (BULK || TLD) ? (double)hc[0] / mx : 0.0);
  cudaFree(d);
  cudaFree(cp);
  cudaFree(src);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, 1>(sms);
  run<256, 1>(sms);
  run<64, 1>(sms);
  run_pair<128>(sms);
  run_pair<256>(sms);
  run<128, 1, true>(sms);
  run_pair<128, true>(sms);
  run<128, 1, false, 16>(sms);
  run<128, 1, false, 0, 4>(sms);
  run<128, 1, false, 0, 1>(sms);
  run<128, 1, false, 0, 32>(sms);
  return 0;
}
