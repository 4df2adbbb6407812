// Microbenchmark: per-SM throughput of fp32 -> int64 round-to-nearest-even
// conversions used by the dW epilogue (cvt.rni.s64.f32 vs alternatives).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_cvt scripts/ubench_cvt.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ long long cvt_s64(float x) { return __float2ll_rn(x); }

// Pure-ALU exact RNE float -> int64 (|x| < 2^62).
__device__ __forceinline__ long long cvt_alu(float x) {
  const uint32_t b = __float_as_uint(x);
  const int e = (int)((b >> 23) & 0xFF);
  const uint32_t m = (b & 0x7FFFFFu) | 0x800000u;
  const int sh = e - 150;
  unsigned long long mag;
  if (sh >= 0) {
    mag = (unsigned long long)m << sh;
  } else {
    const int r = min(-sh, 25);
    const uint32_t half = 1u << (r - 1);
    const uint32_t keep = (r >= 25) ? 0u : (m >> r);
    const uint32_t rem = m & ((1u << r) - 1u);
    const uint32_t up = (rem > half) || (rem == half && (keep & 1u));
    mag = (r >= 25) ? 0ull : (unsigned long long)(keep + up);
  }
  return (b >> 31) ? -(long long)mag : (long long)mag;
}

// Split: |x| < 2^31 via cvt.rni.s32, else exact shift (x is integral there).
__device__ __forceinline__ long long cvt_split(float x) {
  if (fabsf(x) < 2147483648.f) return (long long)__float2int_rn(x);
  const uint32_t b = __float_as_uint(x);
  const int sh = (int)((b >> 23) & 0xFF) - 150;
  const unsigned long long mag = (unsigned long long)((b & 0x7FFFFFu) | 0x800000u) << sh;
  return (b >> 31) ? -(long long)mag : (long long)mag;
}

template <int MODE>
__global__ void k(const float* in, long long* out, int iters, long long* cycles) {
  float v[16];
  for (int j = 0; j < 16; ++j) v[j] = in[(threadIdx.x * 16 + j) & 1023];
  long long acc[16] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = v[j];
      if (MODE == 0) acc[j] += cvt_s64(x);
      if (MODE == 1) acc[j] += (long long)__float2int_rn(x);
      if (MODE == 2) acc[j] += cvt_alu(x);
      if (MODE == 3) acc[j] += cvt_split(x);
      v[j] = __int_as_float(__float_as_int(x) ^ (it & 1));   // defeat hoisting
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  long long s = 0;
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

int main() {
  const int threads = 512, blocks = 148, iters = 2048;
  float h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (i % 3 == 0 ? -1.f : 1.f) * (float)(i * 977 % 100000) * 37.25f * (1 << (i % 20));
  float* din;
  long long *dout, *dcyc;
  cudaMalloc(&din, sizeof(h));
  cudaMalloc(&dout, threads * blocks * 8);
  cudaMalloc(&dcyc, 8);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[4] = {"cvt.rni.s64.f32", "cvt.rni.s32.f32", "alu exact", "s32 + shift"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<blocks, threads>>>(din, dout, iters, dcyc);
      if (mode == 1) k<1><<<blocks, threads>>>(din, dout, iters, dcyc);
      if (mode == 2) k<2><<<blocks, threads>>>(din, dout, iters, dcyc);
      if (mode == 3) k<3><<<blocks, threads>>>(din, dout, iters, dcyc);
    }
    long long cyc;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)threads * iters * 16;   // per SM (one block per SM)
    printf("%-18s %8.2f conversions/clk/SM (+int64 add)\n", names[mode], ops / cyc);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
