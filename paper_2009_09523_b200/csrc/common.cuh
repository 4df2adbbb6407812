// Shared helpers for the B200 virtual-node engine.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace vntb {

// Raised inside the engine and mapped to a VNT_ERR_* status at the C-ABI.
struct EngineError : std::runtime_error {
  int code;
  EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define VNT_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t err__ = (call);                                                         \
    if (err__ != cudaSuccess)                                                           \
      throw ::vntb::EngineError(9, std::string(#call " failed: ") +                     \
                                       cudaGetErrorString(err__) + " at " __FILE__ ":" + \
                                       std::to_string(__LINE__));                       \
  } while (0)

#define VNT_LAUNCH_CHECK() VNT_CUDA(cudaGetLastError())

constexpr int kLossScaleBits = 32;   // default per-row loss quantisation 2^32 (exact int64 sum)
// A virtual node's rows are padded to a multiple of this in a pass (zero
// deltas): its dW K-chain runs in whole k16 steps of kind::f16 (k8 of tf32).
constexpr int kNodeRowPad = 16;

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t round_up(uint64_t a, uint64_t b) { return ceil_div(a, b) * b; }
// smallest k with 2^k >= n (0 for n <= 1)
inline int ceil_log2(uint64_t n) {
  int k = 0;
  while (k < 63 && (1ull << k) < n) ++k;
  return k;
}

// max with NaN propagation (max.NaN.f32): one instruction tracks both a
// range check and a non-finite check.
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Activation codes follow model.hpp:20 (relu, tanh, identity).
__device__ __forceinline__ float act_fwd(int act, float z) {
  if (act == 0) return z > 0.f ? z : 0.f;
  if (act == 1) return tanhf(z);
  return z;
}
// f'(z) expressed through the stored activation a = f(z) (model.cpp:216-228):
// relu'(z) = [z > 0] = [a > 0]; tanh'(z) = 1 - tanh(z)^2 = 1 - a^2.
__device__ __forceinline__ float act_grad_from_out(int act, float a) {
  if (act == 0) return a > 0.f ? 1.f : 0.f;
  if (act == 1) return 1.f - a * a;
  return 1.f;
}

}  // namespace vntb
