// Sharded update of a multi-GPU step.
//
// Each layer's gradient slice [W (in x out, row-major) | b (out)] — contiguous
// in the reference layout — is reduce-scattered in int64 (rank r receives
// elements [r c, (r+1) c) of the slice, c = ceil(n / G) rounded up to 32), so
// a rank updates 1/G of the parameters:
//   k_sgd_shard    exact mean (double(S) 2^-s / B), SGD / momentum on the fp64
//                  master, the new fp32 weights into the all-gather send chunk;
//   k_expand_*     after the all-gather of those chunks: the fp32 copies the
//                  GEMMs read (a tcgen05 layer: W's split-fp16 hi/lo twins;
//                  other layers: W and Wᵀ; the bias),
//                  the same bits the unsharded k_sgd_weight writes.
#pragma once

#include "kernels_simt.cuh"

namespace vntb {

struct ShardSgdArgs {
  const long long* Gs;       // this rank's reduced chunk of the layer slice
  double* w64;               // fp64 master, slice base
  double* v64;               // momentum (slice base) or nullptr
  float* out32;              // this rank's all-gather send chunk
  unsigned long long* gmax;  // [2]: max |g| of the weight and of the bias tensor
  const long long* tail;
  int ntail_flags;
  const StepParams* sp;
  const unsigned long long* h16max;   // see SgdArgs
  int h16n;
  int tw;                    // tensor id of the weight (bias = tw + 1)
  long long lo, hi;          // this rank's slice range
  long long nw;              // weight elements of the slice (in * out)
};

template <bool MOM>
__global__ void __launch_bounds__(256) k_sgd_shard(ShardSgdArgs a) {
  if (block_poisoned(a.tail, a.ntail_flags, a.sp, a.h16max, a.h16n)) return;
  const double inv_b = a.sp->inv_b, lr = a.sp->lr, mu = a.sp->mu;
  const double isw = a.sp->inv_scale[a.tw], isb = a.sp->inv_scale[a.tw + 1];
  double mw = 0.0, mb = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = a.lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.hi; i += stride) {
    const long long k = i - a.lo;
    const bool bias = i >= a.nw;
    // same operation order as k_sgd_weight / k_sgd_twins / sgd_one (bitwise identical update)
    const double g = __dmul_rn(__ll2double_rn(a.Gs[k]) * (bias ? isb : isw), inv_b);
    double u = g;
    if constexpr (MOM) {
      u = __dadd_rn(__dmul_rn(mu, a.v64[i]), g);
      a.v64[i] = u;
    }
    const double w = __dsub_rn(a.w64[i], __dmul_rn(lr, u));
    a.w64[i] = w;
    a.out32[k] = __double2float_rn(w);
    if (bias) mb = fmax(mb, fabs(g));
    else mw = fmax(mw, fabs(g));
  }
  block_max_to(a.gmax, mw);
  __syncthreads();   // block_max_to's smem is reused
  block_max_to(a.gmax + 1, mb);
}

// fp64 slice range -> fp32 (the all-gather send chunk as of the current master).
__global__ void k_f64_to_f32(const double* __restrict__ src, float* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = __double2float_rn(src[i]);
}

// Gathered fp32 weight [rows][cols] -> row-major copy and split-fp16 twins,
// transposed fp32 copy (each output nullable), 32x32 tiles through smem.
// The twins' range flag is tw.flag (kTailH16: these twins feed this step).
__global__ void k_expand_weight(const float* __restrict__ src, int rows, int cols,
                                float* __restrict__ w32, float* __restrict__ wt32, Twin16 tw) {
  __shared__ float tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const float mul = tw.hi ? *tw.mul : 1.f;
  float m = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = r0 + ty + 8 * k, c = c0 + tx;
    float v = 0.f;
    if (r < rows && c < cols) {
      const size_t idx = (size_t)r * cols + c;
      v = src[idx];
      if (w32) w32[idx] = v;
      if (tw.hi) {
        put16(tw.hi, tw.lo, idx, v, mul);
        m = fmax_nan(m, fabsf(v));
      }
    }
    tile[ty + 8 * k][tx] = v;
  }
  if (tw.hi) twin_flush(tw, m, mul);
  if (!wt32) return;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c0 + ty + 8 * k, r = r0 + tx;
    if (r < rows && c < cols) {
      const float v = tile[tx][ty + 8 * k];
      const size_t o = (size_t)c * rows + r;
      wt32[o] = v;
    }
  }
}

__global__ void k_expand_vec(const float* __restrict__ src, int n, float* __restrict__ w32) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) w32[i] = src[i];
}

}  // namespace vntb
