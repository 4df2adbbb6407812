// tcgen05 MMA issue-rate probe: every SM issues R back-to-back MMAs
// (cta_group::1, M=128, N=256) from fixed shared-memory operands into one TMEM
// accumulator; reports dense TFLOP/s for kind::tf32 (K=8 per MMA) and
// kind::f16 (K=16 per MMA).  Operand values are irrelevant to the rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_mma_rate scripts/ubench_mma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
constexpr int M = 128, N = 256;

template <bool F16>
__global__ void __launch_bounds__(128, 1) k_rate(int R, int* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < (M + N) * 128 / 4; i += 128) ((uint32_t*)base)[i] = 0x3c003c00u;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = F16 ? ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24))
                               : ((1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
    const uint64_t ad = sdesc_sw128(su32(base)), bd = sdesc_sw128(su32(base + M * 128));
    for (int i = 0; i < R; ++i) {
      const uint64_t o = (uint64_t)((i & 3) * 2);
      if (F16)
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ad + o), "l"(bd + o), "r"(idesc) : "memory");
      else
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(ad + o), "l"(bd + o), "r"(idesc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  if (tid == 0 && R < 0) *sink = 1;
}

template <bool F16>
void run(int sms) {
  const int smem = (M + N) * 128 + 1024, R = 200000;
  cudaFuncSetAttribute(k_rate<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* sink;
  cudaMalloc(&sink, 4);
  k_rate<F16><<<sms, 128, smem>>>(1000, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_rate<F16><<<sms, 128, smem>>>(R, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * M * N * (F16 ? 16 : 8) * (double)R * sms;
    printf("kind::%s  %d CTAs: %.1f TFLOP/s (%.3f ms) %s\n", F16 ? "f16 " : "tf32", sms, flops / ms / 1e9, ms,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false>(sms);
  run<true>(sms);
  run<false>(sms);
  return 0;
}
