// FFMA / memory-bound kernels of the virtual-node step (sm_100a).
//
// Layout in HBM: for a pass of `rows` rows (virtual nodes
// concatenated in ascending node id, exactly the contiguous slices of
// virtual_exec.cpp:221-238, each node's rows padded to a multiple of 8 with
// pad rows; valid[r] = 0 marks them):
//   X[l]  fp32 [rows][w_l]      activations (X[0] = input), row-major
//   D[l]  fp32 [rows][w_l]      dLoss/dZ_l (l = 1..L), zero on pad rows
//   G     int64 [P + gap + tail] fixed-point gradient sum (exact, order-free)
// The per-node dW GEMMs read X and D as they are (K = rows: MN-major tcgen05
// operands), so no feature-major copies exist.
#pragma once

#include "common.cuh"

namespace vntb {

// Split-fp16 operands of the tcgen05 GEMMs (gemm mode 3XF16): an operand
// tensor x is stored as two fp16 arrays with x 2^sigma ~= hi + lo,
//   hi = fp16_rn(x 2^sigma),  lo = fp16_rn(x 2^sigma - hi)
// (22 significant bits, the fp32 product hi*hi + hi*lo + lo*hi of two such
// operands runs on kind::f16 at twice the kind::tf32 rate).  sigma is one
// power of two per operand tensor, chosen each step from the previous step's
// max|x| over all ranks so that max|x| 2^sigma sits in [2^12, 2^13)
// (DESIGN.md §3): fp16 range limits then cost nothing — an element 2^-38 of
// the tensor max still keeps its absolute error below 2^-25 2^-sigma.
// Producers track max|x| (one atomicMax per warp) and flag |x 2^sigma| >=
// kH16Lim in the tail (kTailH16: the step is redone at the new sigma, the
// update is skipped on device).
constexpr float kH16Lim = 32768.f;
// max|x| 2^sigma below this (global max, sigma below kH16SigMax): the fp16
// split would lose bits to subnormals; the update is skipped and the step
// redone at the retuned sigma (a first step with far-off initial scales).
constexpr float kH16Under = 0.25f;
constexpr int kH16SigMax = 100;
struct Twin16 {
  __half* hi;
  __half* lo;
  const float* mul;            // 2^sigma of the operand (step parameters)
  unsigned long long* amax;    // max |x| of the operand, fp32 bits
  long long* flag;             // tail slot counting |x 2^sigma| >= kH16Lim
};

__device__ __forceinline__ void put16(__half* hi, __half* lo, size_t idx, float v, float mul) {
  const float s = v * mul;   // exact: power of two
  const __half h = __float2half_rn(s);
  hi[idx] = h;
  lo[idx] = __float2half_rn(s - __half2float(h));   // s - h exact in fp32
}

// max |x| of the calling lanes into t.amax (warp reduce, one atomic) and the
// range flag; NaN propagates into the max (its bits order above inf).
__device__ __forceinline__ void twin_flush(const Twin16& t, float m, float mul) {
  const unsigned mask = __activemask();
  const unsigned b = __reduce_max_sync(mask, __float_as_uint(m));
  unsigned lane;
  asm("mov.u32 %0, %%laneid;" : "=r"(lane));
  if (b != 0u && lane == (unsigned)(__ffs(mask) - 1)) {
    // filter on a (possibly stale, never larger) cached copy of the max: most
    // warps skip the same-address atomic, which serialises in L2
    if ((unsigned long long)b > *t.amax) atomicMax(t.amax, (unsigned long long)b);
    if (!(__uint_as_float(b) * mul < kH16Lim)) atomicAdd(reinterpret_cast<unsigned long long*>(t.flag), 1ull);
  }
}

// Tail slots of the int64 accumulator (all summed exactly by the collective).
// kTailLossRange counts rows whose quantised loss could overflow the int64 sum
// (the step is redone at a coarser loss quantum); kTailPartials counts the
// per-node partials of a device_step round (int64 headroom check at sync).
enum : int {
  kTailLoss = 0, kTailExamples = 1, kTailNonfinite = 2, kTailLossRange = 3, kTailPartials = 4,
  kTailH16 = 5,    // an fp16 operand of this step left its range (redo at a new sigma)
  kTailH16W = 6,   // the weight twins written by this step's update left it (re-split)
  kTailOverflow = 7
};

// Per-step values the kernels read from device memory (one small H2D copy per
// step), so the launch sequence of a step is static and can be replayed as a
// CUDA graph while the fixed-point scales adapt.
constexpr int kMaxLayers = 64;
struct StepParams {
  float scale[2 * kMaxLayers];       // 2^s_t: per-node partial quantisation multiplier
  // split-fp16 operand scales 2^sigma / 2^-sigma: X[l] at l, D[l] at L+1+l,
  // the weights (all layers) at 2L+2 (h16_op_*)
  float h16_mul[2 * kMaxLayers + 4];
  float h16_inv[2 * kMaxLayers + 4];
  double inv_scale[2 * kMaxLayers];  // 2^-s_t
  double lr, mu, inv_b;
  double loss_scale;                 // 2^b: per-row loss quantum 2^-b
  double loss_lim;                   // |row loss| * 2^b must stay below this (2^62 / rows bound)
  const double* x;                   // this step's device-resident batch (k_stage_rows)
  const double* y;
};

// ---------------------------------------------------------------- ingest
// fp64 batch rows (reference Batch layout, data.hpp:14-31) -> fp32 X0 and/or
// its split-fp16 twins (X0 null when only the twins are consumed), row stride
// ld; pad rows (valid[r] == 0) become zeros.  One block per row, two
// elements per thread and iteration.
__global__ void __launch_bounds__(128) k_ingest(const double* __restrict__ x, float* __restrict__ X0,
                                                Twin16 tw, const int* __restrict__ valid, int in, int ld) {
  const int r = blockIdx.x;
  const bool ok = valid[r] != 0;
  const double* xr = x + (size_t)r * in;
  const size_t base = (size_t)r * ld;   // ld >= in: the pad columns stay zero
  const float mul = tw.hi ? *tw.mul : 1.f;
  float m = 0.f;
  if ((in & 1) == 0) {
    for (int j = 2 * threadIdx.x; j < in; j += 2 * blockDim.x) {
      double2 d = ok ? __ldg(reinterpret_cast<const double2*>(xr + j)) : make_double2(0.0, 0.0);
      const float2 v = make_float2(__double2float_rn(d.x), __double2float_rn(d.y));
      if (X0) *reinterpret_cast<float2*>(X0 + base + j) = v;
      if (tw.hi) {
        const float2 s = make_float2(v.x * mul, v.y * mul);
        const __half2 h = __floats2half2_rn(s.x, s.y);
        const float2 hf = __half22float2(h);
        *reinterpret_cast<__half2*>(tw.hi + base + j) = h;
        *reinterpret_cast<__half2*>(tw.lo + base + j) = __floats2half2_rn(s.x - hf.x, s.y - hf.y);
        m = fmax_nan(m, fmax_nan(fabsf(v.x), fabsf(v.y)));
      }
    }
  } else {
    for (int j = threadIdx.x; j < in; j += blockDim.x) {
      const float v = ok ? __double2float_rn(xr[j]) : 0.f;
      if (X0) X0[base + j] = v;
      if (tw.hi) {
        put16(tw.hi, tw.lo, base + j, v, mul);
        m = fmax_nan(m, fabsf(v));
      }
    }
  }
  if (tw.hi) twin_flush(tw, m, mul);
}

// ------------------------------------------------------- small copies
// Kernel copies for the per-step control words (step parameters in, tail and
// max|g| out, lineage-stat backups): the host side is pinned, mapped memory,
// so none of them queues on a copy engine behind a large input prefetch.
__global__ void k_copy_words(const unsigned long long* __restrict__ src,
                             unsigned long long* __restrict__ dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

__global__ void k_copy_f64x2(const double* __restrict__ a, double* __restrict__ a_out,
                             const double* __restrict__ b, double* __restrict__ b_out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    a_out[i] = a[i];
    b_out[i] = b[i];
  }
}

// Device-resident batch -> the pass's input buffers, one CTA per node; the
// source pointers come from the step parameters, so a captured step graph
// stages whatever batch the step is given.
__global__ void k_stage_rows(const StepParams* __restrict__ sp, double* __restrict__ xin,
                             double* __restrict__ yin, const int* __restrict__ row0,
                             const int* __restrict__ nrows, const int* __restrict__ src_row, int in,
                             int out) {
  // blockIdx.x = node, blockIdx.y = slice of its (contiguous) rows
  const int k = blockIdx.x;
  const size_t nx = (size_t)nrows[k] * in, ny = (size_t)nrows[k] * out;
  const double* xs = sp->x + (size_t)src_row[k] * in;
  const double* ys = sp->y + (size_t)src_row[k] * out;
  double* xd = xin + (size_t)row0[k] * in;
  double* yd = yin + (size_t)row0[k] * out;
  const size_t stride = (size_t)gridDim.y * blockDim.x;
  const size_t t0 = (size_t)blockIdx.y * blockDim.x + threadIdx.x;
  // 16-byte moves when both ends are 16-byte aligned (even row offsets)
  if ((((uintptr_t)xs | (uintptr_t)xd) & 15) == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(xs);
    double2* d2 = reinterpret_cast<double2*>(xd);
    for (size_t t = t0; t < nx / 2; t += stride) d2[t] = __ldg(s2 + t);
    if ((nx & 1) && t0 == 0) xd[nx - 1] = xs[nx - 1];
  } else {
    for (size_t t = t0; t < nx; t += stride) xd[t] = __ldg(xs + t);
  }
  for (size_t t = t0; t < ny; t += stride) yd[t] = __ldg(ys + t);
}

// One launch for the head of a small-model step (whole-node path): block
// (0,0) copies the step parameters from mapped pinned memory, every block
// zeroes a share of G + tail + max|g| words, and (stage != 0) the device-
// resident batch is staged as in k_stage_rows, with its pointers read straight
// from the mapped parameters.
__global__ void k_step_prologue(const StepParams* __restrict__ host_sp, StepParams* __restrict__ sp,
                                long long* __restrict__ G, size_t nzero, int stage,
                                double* __restrict__ xin, double* __restrict__ yin,
                                const int* __restrict__ row0, const int* __restrict__ nrows,
                                const int* __restrict__ src_row, int in, int out) {
  const int bid = blockIdx.x + blockIdx.y * gridDim.x, nb = gridDim.x * gridDim.y;
  if (bid == 0) {
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(host_sp);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(sp);
    for (int i = threadIdx.x; i < (int)(sizeof(StepParams) / 8); i += blockDim.x) d[i] = s[i];
  }
  for (size_t i = (size_t)bid * blockDim.x + threadIdx.x; i < nzero; i += (size_t)nb * blockDim.x)
    G[i] = 0;
  if (!stage) return;
  const int k = blockIdx.x;
  const double* xsrc = host_sp->x;
  const double* ysrc = host_sp->y;
  const size_t nx = (size_t)nrows[k] * in, ny = (size_t)nrows[k] * out;
  const double* xs = xsrc + (size_t)src_row[k] * in;
  const double* ys = ysrc + (size_t)src_row[k] * out;
  double* xd = xin + (size_t)row0[k] * in;
  double* yd = yin + (size_t)row0[k] * out;
  const size_t stride = (size_t)gridDim.y * blockDim.x;
  const size_t t0 = (size_t)blockIdx.y * blockDim.x + threadIdx.x;
  for (size_t t = t0; t < nx; t += stride) xd[t] = __ldg(xs + t);
  for (size_t t = t0; t < ny; t += stride) yd[t] = __ldg(ys + t);
}

// ------------------------------------------------------------ input stats
// LayerStats::observe batch part (model.cpp:101-121): per node, per feature,
// sequential fp64 sums in row order; __d*_rn forbid FMA contraction so the
// result is bit-identical to the reference's x86-64 build.
// One feature j of one node (rows r0..r0+n-1 of x): fp64 mean and M2 in row order.
__device__ __forceinline__ void node_feature_stats(const double* __restrict__ x, int in, int r0,
                                                   int n, int j, double* mean, double* m2) {
  const double* xp = x + (size_t)r0 * in + j;
  double m = 0.0;
  int r = 0;
  for (; r + 8 <= n; r += 8) {   // 8 loads in flight, adds in row order
    double t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = __ldg(xp + (size_t)(r + q) * in);
#pragma unroll
    for (int q = 0; q < 8; ++q) m = __dadd_rn(m, t[q]);
  }
  for (; r < n; ++r) m = __dadd_rn(m, __ldg(xp + (size_t)r * in));
  m = __ddiv_rn(m, (double)n);
  double s = 0.0;
  r = 0;
  for (; r + 8 <= n; r += 8) {
    double t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = __ldg(xp + (size_t)(r + q) * in);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double d = __dsub_rn(t[q], m);
      s = __dadd_rn(s, __dmul_rn(d, d));
    }
  }
  for (; r < n; ++r) {
    const double d = __dsub_rn(__ldg(xp + (size_t)r * in), m);
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
  *mean = m;
  *m2 = s;
}

__global__ void k_vn_stats(const double* __restrict__ x, int in, const int* __restrict__ vn_row0,
                           const int* __restrict__ vn_rows, double* __restrict__ vn_mean,
                           double* __restrict__ vn_m2) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (j >= in) return;
  node_feature_stats(x, in, vn_row0[k], vn_rows[k], j, &vn_mean[(size_t)k * in + j],
                     &vn_m2[(size_t)k * in + j]);
}

// LayerStats::combine (model.cpp:123-139) of a device's nodes, ascending id.
// The count arithmetic is done on the host with the same double ops; f1 =
// count*other.count/n and f2 = other.count/n arrive precomputed.
struct CombineStep {
  int vn;        // index into the pass's node table
  int copy;      // lineage empty: *this = other
  double f1, f2;
};

// One feature j: fold nsteps node stats into (mean, m2) in step order; 8 steps'
// loads in flight.  __ldcg: the node stats may come from other CTAs of the
// same launch (k_node_step's last CTA).
__device__ __forceinline__ void combine_feature(double* __restrict__ mean, double* __restrict__ m2,
                                                int in, int j, const double* vn_mean,
                                                const double* vn_m2, const CombineStep* steps,
                                                int nsteps) {
  double mu = mean[j], s = m2[j];
  for (int t0 = 0; t0 < nsteps; t0 += 8) {
    const int tn = min(8, nsteps - t0);
    CombineStep st[8];
    double om[8], os[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < tn) st[q] = steps[t0 + q];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < tn) {
        om[q] = __ldcg(vn_mean + (size_t)st[q].vn * in + j);
        os[q] = __ldcg(vn_m2 + (size_t)st[q].vn * in + j);
      }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q >= tn) break;
      if (st[q].copy) {
        mu = om[q];
        s = os[q];
      } else {
        const double delta = __dsub_rn(om[q], mu);
        s = __dadd_rn(s, __dadd_rn(os[q], __dmul_rn(__dmul_rn(delta, delta), st[q].f1)));
        mu = __dadd_rn(mu, __dmul_rn(delta, st[q].f2));
      }
    }
  }
  mean[j] = mu;
  m2[j] = s;
}

// `steps` may live in pinned host memory (read over the bus): each block first
// copies a chunk of them into shared memory with all threads at once.
__global__ void k_stats_combine(double* __restrict__ mean, double* __restrict__ m2, int in,
                                const double* __restrict__ vn_mean,
                                const double* __restrict__ vn_m2,
                                const CombineStep* __restrict__ steps, int nsteps) {
  constexpr int kChunk = 256;
  __shared__ CombineStep st[kChunk];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  for (int t0 = 0; t0 < nsteps; t0 += kChunk) {
    const int tn = min(kChunk, nsteps - t0);
    __syncthreads();
    for (int t = threadIdx.x; t < tn; t += blockDim.x) st[t] = steps[t0 + t];
    __syncthreads();
    if (j < in) combine_feature(mean, m2, in, j, vn_mean, vn_m2, st, tn);
  }
}

// ------------------------------------------------------ FFMA dense layer
// C[r][n] = init[n] + sum_k A[r][k] * B[k][n] with k strictly ascending in a
// single fmaf chain per output (model.cpp:280-283: z = b; z += a_i * w_io), so
// each output depends only on its row and the weights — never on how many
// rows (virtual nodes) share the launch.  Epilogues:
//   kEpiHidden: a = f(z) -> X[l+1], XT[l+1]
//   kEpiLogits: z -> logits
//   kEpiBwd:    d = z * f'(X[l]) -> D[l], DT[l]   (model.cpp:328-337)
enum : int { kEpiHidden = 0, kEpiLogits = 1, kEpiBwd = 2 };

template <int EPI>
__global__ void __launch_bounds__(256) k_gemm_ffma(
    const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb, int M, int N,
    int K, const float* __restrict__ bias, int act, float* __restrict__ out, int ldo,
    const float* __restrict__ Xprev, int ldx) {
  __shared__ __align__(16) float As[16][64 + 4];
  __shared__ __align__(16) float Bs[16][64 + 4];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int n = n0 + tx * 4 + j;
    const float b0 = (EPI != kEpiBwd && n < N) ? bias[n] : 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = b0;
  }
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = t + e * 256;
      const int mm = idx / 16, kk = idx % 16;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gm * lda + gk] : 0.f;
      const int kb = idx / 64, nn = idx % 64;
      const int gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < N && gkb < K) ? B[(size_t)gkb * ldb + gn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (EPI == kEpiHidden) {
        v = act_fwd(act, v);
      } else if (EPI == kEpiBwd) {
        v = v * act_grad_from_out(act, Xprev[(size_t)r * ldx + n]);
      }
      out[(size_t)r * ldo + n] = v;
    }
  }
}

// One row's loss into the exact int64 loss sum: q = rint(loss * 2^b).  Rows
// outside the range that keeps any sum of the step's rows in int64 are
// counted (kTailLossRange) instead, and the host redoes the step with a
// coarser quantum; non-finite rows are counted as such.
__device__ __forceinline__ bool row_loss_q(double loss, const StepParams* sp, long long* tail,
                                           long long& q) {
  if (!isfinite(loss)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailNonfinite]), 1ull);
    return false;
  }
  const double v = loss * sp->loss_scale;
  if (!(fabs(v) < sp->loss_lim)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailLossRange]), 1ull);
    return false;
  }
  q = __double2ll_rn(v);
  return true;
}

// ------------------------------------------------------------- loss/delta
// model.cpp:289-315, one warp per row, fp64 from fp32 logits.  Row loss is
// quantised at 2^-32 and summed exactly (int64 atomics: order-free).
__global__ void k_loss(const float* __restrict__ logits, const double* __restrict__ y, int rows,
                       int outw, int loss_kind, float* __restrict__ D,
                       const int* __restrict__ valid, long long* __restrict__ tail,
                       const StepParams* __restrict__ sp) {
  __shared__ unsigned long long block_loss;   // exact int64 sum of this block's rows
  if (threadIdx.x == 0) block_loss = 0;
  __syncthreads();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int r = warp;
  if (warp < rows && !valid[r]) {   // pad row: zero delta, no loss
    for (int o = lane; o < outw; o += 32) D[(size_t)r * outw + o] = 0.f;
  } else if (warp < rows) {
    const float* z = logits + (size_t)r * outw;
    const double* yr = y + (size_t)r * outw;
    double loss = 0.0;
    if (loss_kind == 0) {
      for (int o = lane; o < outw; o += 32) {
        const double d = (double)z[o] - yr[o];
        loss += d * d;
        D[(size_t)r * outw + o] = (float)(2.0 * d / (double)outw);
      }
#pragma unroll
      for (int s = 16; s; s >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, s);
      loss /= (double)outw;
    } else {
      double mx = -1e300;
      for (int o = lane; o < outw; o += 32) mx = fmax(mx, (double)z[o]);
#pragma unroll
      for (int s = 16; s; s >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, s));
      double norm = 0.0;
      for (int o = lane; o < outw; o += 32) norm += exp((double)z[o] - mx);
#pragma unroll
      for (int s = 16; s; s >>= 1) norm += __shfl_xor_sync(0xffffffffu, norm, s);
      const double lognorm = log(norm);
      for (int o = lane; o < outw; o += 32) {
        const double zm = (double)z[o] - mx;
        loss -= yr[o] * (zm - lognorm);
        D[(size_t)r * outw + o] = (float)(exp(zm) / norm - yr[o]);
      }
#pragma unroll
      for (int s = 16; s; s >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, s);
    }
    long long q;
    if (lane == 0 && row_loss_q(loss, sp, tail, q))
      atomicAdd(&block_loss, (unsigned long long)q);   // shared memory, order-free
  }
  __syncthreads();
  if (threadIdx.x == 0 && block_loss)
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailLoss]), block_loss);
}

// Fixed-point quantisation of one per-node partial:
// q = rint(g * 2^s).  |g * 2^s| must stay below lim = 2^62 / V so that any sum
// of V partials fits int64; violations are counted and force a re-scaled redo.
__device__ __forceinline__ long long quantise(float g, float scale, float lim,
                                              long long* __restrict__ tail, int tensor) {
  const float v = g * scale;
  if (!isfinite(v)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailNonfinite]), 1ull);
    return 0;
  }
  if (fabsf(v) >= lim) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailOverflow + tensor]), 1ull);
    return 0;
  }
  return __float2ll_rn(v);
}

// ------------------------------------------------ per-node dW, FFMA path
// g_k[i][o] = sum_{r in node k} X[r][i] * D[r][o] (one fmaf chain, rows
// ascending); blockIdx.z = node.  Quantised per node and added with exact
// int64 atomics into the zeroed weight slice of G (order-free).
__global__ void __launch_bounds__(256) k_dw_ffma(
    const float* __restrict__ X, const float* __restrict__ D, int in, int out,
    const int* __restrict__ vn_row0, const int* __restrict__ vn_rows,
    const float* __restrict__ scale_p, float lim, long long* __restrict__ G,
    long long* __restrict__ tail, int tensor) {
  __shared__ __align__(16) float As[16][64 + 4];
  __shared__ __align__(16) float Bs[16][64 + 4];
  const float scale = *scale_p;
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int i0 = blockIdx.y * 64, o0 = blockIdx.x * 64;
  const int v = blockIdx.z;
  const int r0 = vn_row0[v], n = vn_rows[v];
  float g[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) g[i][j] = 0.f;
  for (int k0 = 0; k0 < n; k0 += 16) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {   // rows of X / D, features contiguous across lanes
      const int idx = t + e * 256;
      const int mm = idx % 64, kk = idx / 64;
      const bool kin = (k0 + kk) < n;
      const size_t r = (size_t)(r0 + k0 + kk);
      As[kk][mm] = (kin && i0 + mm < in) ? X[r * in + i0 + mm] : 0.f;
      Bs[kk][mm] = (kin && o0 + mm < out) ? D[r * out + o0 + mm] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) g[i][j] = fmaf(a[i], b[j], g[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = i0 + ty * 4 + i;
    if (gi >= in) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int go = o0 + tx * 4 + j;
      if (go >= out) continue;
      const long long q = quantise(g[i][j], scale, lim, tail, tensor);
      if (q) atomicAdd(reinterpret_cast<unsigned long long*>(G + (size_t)gi * out + go),
                       (unsigned long long)q);
    }
  }
}

// Per-node bias gradient (model.cpp:322: gb = delta): column sums of D over
// the node's rows, fp32 in row order, quantised per node; one CTA column per
// node, exact int64 atomics (order-free) into the zeroed bias slice of G.
// D is either fp32 (Dh == nullptr) or given only as its split-fp16 twins:
// d = (hi + lo) 2^-sigma (hi + lo exact in fp32, the scaling exact).
__global__ void k_db(const float* __restrict__ D, const __half* __restrict__ Dh,
                     const __half* __restrict__ Dl, const float* __restrict__ inv_p, int out,
                     const int* __restrict__ vn_row0, const int* __restrict__ vn_rows,
                     const float* __restrict__ scale_p, float lim, long long* __restrict__ G,
                     long long* __restrict__ tail, int tensor) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (o >= out) return;
  const int r0 = vn_row0[v], n = vn_rows[v];
  const float scale = *scale_p;
  float g = 0.f;
  int r = 0;
  if (Dh) {
    const float inv = *inv_p;
    const __half* dh = Dh + (size_t)r0 * out + o;
    const __half* dl = Dl + (size_t)r0 * out + o;
    for (; r + 8 <= n; r += 8) {   // 8 loads in flight, adds still in row order
      float t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        t[j] = (__half2float(dh[(size_t)(r + j) * out]) + __half2float(dl[(size_t)(r + j) * out])) * inv;
#pragma unroll
      for (int j = 0; j < 8; ++j) g += t[j];
    }
    for (; r < n; ++r) g += (__half2float(dh[(size_t)r * out]) + __half2float(dl[(size_t)r * out])) * inv;
  } else {
    const float* d = D + (size_t)r0 * out + o;
    for (; r + 8 <= n; r += 8) {
      float t[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] = __ldg(d + (size_t)(r + j) * out);
#pragma unroll
      for (int j = 0; j < 8; ++j) g += t[j];
    }
    for (; r < n; ++r) g += __ldg(d + (size_t)r * out);
  }
  const long long q = quantise(g, scale, lim, tail, tensor);
  if (q) atomicAdd(reinterpret_cast<unsigned long long*>(&G[o]), (unsigned long long)q);
}

// k_db on the split-fp16 twins, two columns per thread (__half2 loads: 128 B
// per warp and row): the same per-column row order as k_db, so the same bits.
__global__ void k_db2(const __half* __restrict__ Dh, const __half* __restrict__ Dl,
                      const float* __restrict__ inv_p, int out, const int* __restrict__ vn_row0,
                      const int* __restrict__ vn_rows, const float* __restrict__ scale_p, float lim,
                      long long* __restrict__ G, long long* __restrict__ tail, int tensor) {
  const int o = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int v = blockIdx.y;
  if (o >= out) return;
  const int r0 = vn_row0[v], n = vn_rows[v];
  const float scale = *scale_p, inv = *inv_p;
  const __half2* dh = reinterpret_cast<const __half2*>(Dh + (size_t)r0 * out + o);
  const __half2* dl = reinterpret_cast<const __half2*>(Dl + (size_t)r0 * out + o);
  const size_t ld = (size_t)out / 2;
  float g0 = 0.f, g1 = 0.f;
  int r = 0;
  for (; r + 16 <= n; r += 16) {   // 16 rows in flight, adds in row order per column
    __half2 hh[16], ll[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      hh[j] = dh[(size_t)(r + j) * ld];
      ll[j] = dl[(size_t)(r + j) * ld];
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 h = __half22float2(hh[j]), l = __half22float2(ll[j]);
      g0 += (h.x + l.x) * inv;
      g1 += (h.y + l.y) * inv;
    }
  }
  for (; r < n; ++r) {
    const float2 h = __half22float2(dh[(size_t)r * ld]);
    const float2 l = __half22float2(dl[(size_t)r * ld]);
    g0 += (h.x + l.x) * inv;
    g1 += (h.y + l.y) * inv;
  }
  const long long q0 = quantise(g0, scale, lim, tail, tensor);
  const long long q1 = quantise(g1, scale, lim, tail, tensor);
  if (q0) atomicAdd(reinterpret_cast<unsigned long long*>(&G[o]), (unsigned long long)q0);
  if (q1) atomicAdd(reinterpret_cast<unsigned long long*>(&G[o + 1]), (unsigned long long)q1);
}

// ---------------------------------------------- skinny layers (out <= 32)
template <int NO>   // rows per warp in k_fwd_skinny (R*NO accumulators per lane)
__host__ __device__ constexpr int skinny_rows() { return NO > 16 ? 2 : 4; }
// Forward with few outputs (the 4096 -> 10 classifier): one warp per row,
// lane-strided partial dot products over k then a fixed xor tree, so every
// output depends only on its row.
template <int NO>
__global__ void __launch_bounds__(256) k_fwd_skinny(const float* __restrict__ X, int K,
                                                    const float* __restrict__ WT, int no,
                                                    const float* __restrict__ bias, int rows,
                                                    int act, int last, float* __restrict__ out) {
  // A warp owns R rows so each W value read serves all of them; W^T is staged
  // through shared memory in k-chunks ([o][k], conflict-free).  Per (row, o)
  // the partial sums run lane-strided over k in ascending order and meet in a
  // fixed xor tree, so every output depends only on its row.
  constexpr int R = skinny_rows<NO>();
  constexpr int KC = 8192 / NO;   // 32 KB of W^T per chunk
  __shared__ float ws[NO][KC];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int row0 = warp * R;
  const float* x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) x[r] = X + (size_t)min(row0 + r, rows - 1) * K;
  float acc[R][NO];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int o = 0; o < NO; ++o) acc[r][o] = 0.f;
  for (int k0 = 0; k0 < K; k0 += KC) {
    const int kn = min(KC, K - k0);
    __syncthreads();
    for (int t = threadIdx.x; t < NO * KC; t += blockDim.x) {
      const int o = t / KC, kk = t % KC;
      ws[o][kk] = (o < no && kk < kn) ? __ldg(WT + (size_t)o * K + k0 + kk) : 0.f;
    }
    __syncthreads();
    if (row0 < rows) {
#pragma unroll 4
      for (int kk = lane; kk < kn; kk += 32) {
        float a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = __ldg(x[r] + k0 + kk);
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          if (o < no) {
            const float wo = ws[o][kk];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r][o] = fmaf(a[r], wo, acc[r][o]);
          }
        }
      }
    }
  }
  if (row0 >= rows) return;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int o = 0; o < NO; ++o) {
#pragma unroll
      for (int s = 16; s; s >>= 1) acc[r][o] += __shfl_xor_sync(0xffffffffu, acc[r][o], s);
    }
  if (lane < no) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = row0 + r;
      if (row >= rows) break;
      float v = 0.f;
#pragma unroll
      for (int o = 0; o < NO; ++o)
        if (o == lane) v = acc[r][o];
      v += bias[lane];
      if (!last) v = act_fwd(act, v);
      out[(size_t)row * no + lane] = v;
    }
  }
}

// bwd-data through a skinny layer: D[r][i] = (sum_o Dn[r][o] W[i][o]) f'(X[r][i]),
// o ascending; 32 features x chunks*32 rows per block (the row block's Dn
// rows staged in smem), D and/or its split-fp16 twins written row-major.
template <int NO>
__global__ void __launch_bounds__(256) k_bwd_skinny(const float* __restrict__ Dn,
                                                    const float* __restrict__ W, int no, int in,
                                                    int rows, int act,
                                                    const float* __restrict__ Xprev,
                                                    float* __restrict__ Dout, Twin16 tw,
                                                    int chunks) {
  const float mul = tw.hi ? *tw.mul : 1.f;
  float m = 0.f;
  __shared__ float dn[32][NO];
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const int i = blockIdx.x * 32 + tx;
  float w[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) w[o] = (i < in && o < no) ? W[(size_t)i * no + o] : 0.f;
  for (int chunk = 0; chunk < chunks; ++chunk) {
    const int r0 = (blockIdx.y * chunks + chunk) * 32;
    if (r0 >= rows) break;
    __syncthreads();
    for (int k = ty * 32 + tx; k < 32 * NO; k += 256) {
      const int rr = k / NO, o = k % NO;
      dn[rr][o] = (r0 + rr < rows && o < no) ? Dn[(size_t)(r0 + rr) * no + o] : 0.f;
    }
    __syncthreads();
    if (i >= in) continue;
#pragma unroll 4
    for (int k = ty; k < 32; k += 8) {
      const int r = r0 + k;
      if (r >= rows) break;
      float acc = 0.f;
#pragma unroll
      for (int o = 0; o < NO; ++o) acc = fmaf(dn[k][o], w[o], acc);
      const size_t idx = (size_t)r * in + i;
      const float v = acc * act_grad_from_out(act, Xprev[idx]);
      if (Dout) Dout[idx] = v;
      if (tw.hi) {
        put16(tw.hi, tw.lo, idx, v, mul);
        m = fmax_nan(m, fabsf(v));
      }
    }
  }
  if (tw.hi) twin_flush(tw, m, mul);
}

// Per-node dW of a skinny layer: thread per input feature i, NO accumulators,
// rows of the node in order; node partials quantised and added with int64
// atomics (exact) into the zeroed weight slice of G.
template <int NO>
__global__ void k_dw_skinny(const float* __restrict__ X, int in, const float* __restrict__ Dn,
                            int no,
                            const int* __restrict__ vn_row0, const int* __restrict__ vn_rows,
                            const float* __restrict__ scale_p, float lim,
                            long long* __restrict__ G, long long* __restrict__ tail, int tensor) {
  static_assert(NO % 4 == 0, "dn rows are read as float4");
  __shared__ __align__(16) float dn[64][NO];
  const float scale = *scale_p;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  const int r0 = vn_row0[v], n = vn_rows[v];
  float g[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) g[o] = 0.f;
  for (int c = 0; c < n; c += 64) {
    const int cn = min(64, n - c);
    __syncthreads();
    for (int k = threadIdx.x; k < cn * NO; k += blockDim.x)
      dn[k / NO][k % NO] = (k % NO < no) ? Dn[(size_t)(r0 + c + k / NO) * no + k % NO] : 0.f;
    __syncthreads();
    if (i < in) {
      const float* xp = X + (size_t)(r0 + c) * in + i;
      int rr = 0;
      for (; rr + 8 <= cn; rr += 8) {   // 8 loads in flight, FMAs in row order
        float a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = __ldg(xp + (size_t)(rr + j) * in);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4* d4 = reinterpret_cast<const float4*>(&dn[rr + j][0]);
#pragma unroll
          for (int o = 0; o < NO; o += 4) {   // broadcast float4 reads: 4x fewer LDS
            const float4 d = d4[o / 4];
            g[o] = fmaf(a[j], d.x, g[o]);
            g[o + 1] = fmaf(a[j], d.y, g[o + 1]);
            g[o + 2] = fmaf(a[j], d.z, g[o + 2]);
            g[o + 3] = fmaf(a[j], d.w, g[o + 3]);
          }
        }
      }
      for (; rr < cn; ++rr) {
        const float a = __ldg(xp + (size_t)rr * in);
#pragma unroll
        for (int o = 0; o < NO; ++o) g[o] = fmaf(a, dn[rr][o], g[o]);
      }
    }
  }
  if (i >= in) return;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (o >= no) break;
    const long long q = quantise(g[o], scale, lim, tail, tensor);
    if (q) atomicAdd(reinterpret_cast<unsigned long long*>(&G[(size_t)i * no + o]),
                     (unsigned long long)q);
  }
}

// Forward of a skinny layer with all of W^T ([no][K], K % 4 == 0) resident in
// shared memory: a persistent grid; a warp takes 4 rows at a time so every W
// value read from smem serves 4 rows (smem bandwidth, not HBM, bound the
// one-row version), float4 loads of the rows (2 per row in flight per lane);
// per (row, output) the lane-strided partial sums run over k ascending, then a
// fixed xor tree, so every output depends only on its row.
template <int NO>
__global__ void __launch_bounds__(512) k_fwd_skinny_res(const float* __restrict__ X, int K,
                                                        const float* __restrict__ WT, int no,
                                                        const float* __restrict__ bias, int rows,
                                                        int act, int last, float* __restrict__ out) {
  constexpr int R = 4;
  extern __shared__ float4 wsm[];
  const int K4 = K >> 2;
  for (int i = threadIdx.x; i < no * K4; i += blockDim.x) wsm[i] = __ldg(reinterpret_cast<const float4*>(WT) + i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * R; r0 < rows; r0 += nw * R) {
    const float4* xr[R];
#pragma unroll
    for (int q = 0; q < R; ++q) xr[q] = reinterpret_cast<const float4*>(X + (size_t)min(r0 + q, rows - 1) * K);
    float acc[R][NO];
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int o = 0; o < NO; ++o) acc[q][o] = 0.f;
    auto fold = [&](const float4 (&xv)[R], int k4) {
#pragma unroll
      for (int o = 0; o < NO; ++o)
        if (o < no) {
          const float4 w = wsm[o * K4 + k4];
#pragma unroll
          for (int q = 0; q < R; ++q) {
            acc[q][o] = fmaf(xv[q].x, w.x, acc[q][o]);
            acc[q][o] = fmaf(xv[q].y, w.y, acc[q][o]);
            acc[q][o] = fmaf(xv[q].z, w.z, acc[q][o]);
            acc[q][o] = fmaf(xv[q].w, w.w, acc[q][o]);
          }
        }
    };
    int k4 = lane;
    for (; k4 + 32 < K4; k4 += 64) {   // k ascending per lane: k4, k4 + 32
      float4 xa[R], xb[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        xa[q] = __ldg(xr[q] + k4);
        xb[q] = __ldg(xr[q] + k4 + 32);
      }
      fold(xa, k4);
      fold(xb, k4 + 32);
    }
    for (; k4 < K4; k4 += 32) {
      float4 xa[R];
#pragma unroll
      for (int q = 0; q < R; ++q) xa[q] = __ldg(xr[q] + k4);
      fold(xa, k4);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
#pragma unroll
      for (int o = 0; o < NO; ++o) {
#pragma unroll
        for (int sft = 16; sft; sft >>= 1) acc[q][o] += __shfl_xor_sync(0xffffffffu, acc[q][o], sft);
      }
      float v = 0.f;
#pragma unroll
      for (int o = 0; o < NO; ++o)
        if (o == lane) v = acc[q][o];
      if (lane < no && r0 + q < rows) {
        v += bias[lane];
        if (!last) v = act_fwd(act, v);
        out[(size_t)(r0 + q) * no + lane] = v;
      }
    }
  }
}

// Backward through a skinny layer l (no <= 32 outputs) for one virtual node and
// a slab of 128 input features per block (thread = feature i), over the
// node's rows in order — one read of X[l] for three results:
//   dW_l[i][o]  = sum_r X[r][i] Dn[r][o]             (fmaf chain, rows ascending)
//   D[l][r][i]  = (sum_o Dn[r][o] W[i][o]) f'(X[r][i]) (o ascending)
//   db_{l-1}[i] = sum_r D[l][r][i]                    (rows ascending)
// the same operation orders as k_dw_skinny, k_bwd_skinny and k_db.  Node
// partials are quantised and added into G with int64 atomics (exact).  D[l]
// is written as the split-fp16 twins and/or plain (each nullable); Gb == nullptr
// (l == 0): no bwd-data / db.
template <int NO>
__global__ void __launch_bounds__(128) k_skinny_backward(
    const float* __restrict__ X, const float* __restrict__ Dn, const float* __restrict__ W, int in, int no,
    int act, const int* __restrict__ vn_row0, const int* __restrict__ vn_rows, float* __restrict__ Dout,
    Twin16 twd, const float* __restrict__ scale_w, long long* __restrict__ Gw, int tw,
    const float* __restrict__ scale_b, long long* __restrict__ Gb, int tb, float lim,
    long long* __restrict__ tail) {
  static_assert(NO % 4 == 0, "dn rows are read as float4");
  __shared__ __align__(16) float dn[64][NO];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  const int r0 = vn_row0[v], n = vn_rows[v];
  const bool data = Gb != nullptr;
  const float mul = twd.hi ? *twd.mul : 1.f;
  float m = 0.f;
  float w[NO], g[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    w[o] = (data && i < in && o < no) ? __ldg(W + (size_t)i * no + o) : 0.f;
    g[o] = 0.f;
  }
  float db = 0.f;
  for (int c = 0; c < n; c += 64) {
    const int cn = min(64, n - c);
    __syncthreads();
    for (int k = threadIdx.x; k < cn * NO; k += blockDim.x)
      dn[k / NO][k % NO] = (k % NO < no) ? Dn[(size_t)(r0 + c + k / NO) * no + k % NO] : 0.f;
    __syncthreads();
    if (i >= in) continue;
    const float* xp = X + (size_t)(r0 + c) * in + i;
    // the next 8 rows are loaded while these 8 are folded (16 loads in flight)
    float an[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) an[j] = j < cn ? __ldg(xp + (size_t)j * in) : 0.f;
    for (int rr = 0; rr < cn; rr += 8) {
      float a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = an[j];
#pragma unroll
      for (int j = 0; j < 8; ++j) an[j] = rr + 8 + j < cn ? __ldg(xp + (size_t)(rr + 8 + j) * in) : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (rr + j >= cn) break;
        const float4* d4 = reinterpret_cast<const float4*>(&dn[rr + j][0]);
        float acc = 0.f;
#pragma unroll
        for (int o = 0; o < NO; o += 4) {
          const float4 d = d4[o / 4];
          g[o] = fmaf(a[j], d.x, g[o]);
          g[o + 1] = fmaf(a[j], d.y, g[o + 1]);
          g[o + 2] = fmaf(a[j], d.z, g[o + 2]);
          g[o + 3] = fmaf(a[j], d.w, g[o + 3]);
          acc = fmaf(d.x, w[o], acc);
          acc = fmaf(d.y, w[o + 1], acc);
          acc = fmaf(d.z, w[o + 2], acc);
          acc = fmaf(d.w, w[o + 3], acc);
        }
        if (data) {
          const float dv = acc * act_grad_from_out(act, a[j]);
          const size_t idx = (size_t)(r0 + c + rr + j) * in + i;
          if (Dout) Dout[idx] = dv;
          if (twd.hi) {
            put16(twd.hi, twd.lo, idx, dv, mul);
            m = fmax_nan(m, fabsf(dv));
          }
          db += dv;
        }
      }
    }
  }
  if (twd.hi) twin_flush(twd, m, mul);
  if (i >= in) return;
  if (data)   // the node's pad rows (up to kNodeRowPad) carry zero deltas
    for (int r = n; r < (int)round_up(n, kNodeRowPad); ++r) {
      const size_t idx = (size_t)(r0 + r) * in + i;
      if (Dout) Dout[idx] = 0.f;
      if (twd.hi) {
        twd.hi[idx] = __float2half_rn(0.f);
        twd.lo[idx] = __float2half_rn(0.f);
      }
    }
  const float sw = *scale_w;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (o >= no) break;
    const long long q = quantise(g[o], sw, lim, tail, tw);
    if (q) atomicAdd(reinterpret_cast<unsigned long long*>(&Gw[(size_t)i * no + o]), (unsigned long long)q);
  }
  if (data) {
    const long long q = quantise(db, *scale_b, lim, tail, tb);
    if (q) atomicAdd(reinterpret_cast<unsigned long long*>(&Gb[i]), (unsigned long long)q);
  }
}

// k_skinny_backward with two adjacent input features per thread (in even):
// float2 loads of X, the D twins as half2, the dn rows read once for both —
// the same per-feature operation order, so the same bits.
template <int NO>
__global__ void __launch_bounds__(128) k_skinny_backward2(
    const float* __restrict__ X, const float* __restrict__ Dn, const float* __restrict__ W, int in, int no,
    int act, const int* __restrict__ vn_row0, const int* __restrict__ vn_rows, float* __restrict__ Dout,
    Twin16 twd, const float* __restrict__ scale_w, long long* __restrict__ Gw, int tw,
    const float* __restrict__ scale_b, long long* __restrict__ Gb, int tb, float lim,
    long long* __restrict__ tail) {
  static_assert(NO % 4 == 0, "dn rows are read as float4");
  __shared__ __align__(16) float dn[64][NO];
  const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int v = blockIdx.y;
  const int r0 = vn_row0[v], n = vn_rows[v];
  const bool data = Gb != nullptr;
  const float mul = twd.hi ? *twd.mul : 1.f;
  float m = 0.f;
  float w0[NO], w1[NO], g0[NO], g1[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const bool ok = data && i < in && o < no;
    w0[o] = ok ? __ldg(W + (size_t)i * no + o) : 0.f;
    w1[o] = ok ? __ldg(W + (size_t)(i + 1) * no + o) : 0.f;
    g0[o] = g1[o] = 0.f;
  }
  float db0 = 0.f, db1 = 0.f;
  for (int c = 0; c < n; c += 64) {
    const int cn = min(64, n - c);
    __syncthreads();
    for (int k = threadIdx.x; k < cn * NO; k += blockDim.x)
      dn[k / NO][k % NO] = (k % NO < no) ? Dn[(size_t)(r0 + c + k / NO) * no + k % NO] : 0.f;
    __syncthreads();
    if (i >= in) continue;
    const float2* xp = reinterpret_cast<const float2*>(X + (size_t)(r0 + c) * in + i);
    const size_t ld2 = (size_t)in / 2;
    float2 an[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) an[j] = j < cn ? __ldg(xp + (size_t)j * ld2) : make_float2(0.f, 0.f);
    for (int rr = 0; rr < cn; rr += 8) {
      float2 a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = an[j];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        an[j] = rr + 8 + j < cn ? __ldg(xp + (size_t)(rr + 8 + j) * ld2) : make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (rr + j >= cn) break;
        const float4* d4 = reinterpret_cast<const float4*>(&dn[rr + j][0]);
        float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
        for (int o = 0; o < NO; o += 4) {
          const float4 d = d4[o / 4];
          g0[o] = fmaf(a[j].x, d.x, g0[o]);
          g0[o + 1] = fmaf(a[j].x, d.y, g0[o + 1]);
          g0[o + 2] = fmaf(a[j].x, d.z, g0[o + 2]);
          g0[o + 3] = fmaf(a[j].x, d.w, g0[o + 3]);
          g1[o] = fmaf(a[j].y, d.x, g1[o]);
          g1[o + 1] = fmaf(a[j].y, d.y, g1[o + 1]);
          g1[o + 2] = fmaf(a[j].y, d.z, g1[o + 2]);
          g1[o + 3] = fmaf(a[j].y, d.w, g1[o + 3]);
          acc0 = fmaf(d.x, w0[o], acc0);
          acc0 = fmaf(d.y, w0[o + 1], acc0);
          acc0 = fmaf(d.z, w0[o + 2], acc0);
          acc0 = fmaf(d.w, w0[o + 3], acc0);
          acc1 = fmaf(d.x, w1[o], acc1);
          acc1 = fmaf(d.y, w1[o + 1], acc1);
          acc1 = fmaf(d.z, w1[o + 2], acc1);
          acc1 = fmaf(d.w, w1[o + 3], acc1);
        }
        if (data) {
          const float dv0 = acc0 * act_grad_from_out(act, a[j].x);
          const float dv1 = acc1 * act_grad_from_out(act, a[j].y);
          const size_t idx = (size_t)(r0 + c + rr + j) * in + i;
          if (Dout) *reinterpret_cast<float2*>(Dout + idx) = make_float2(dv0, dv1);
          if (twd.hi) {
            const float s0 = dv0 * mul, s1 = dv1 * mul;
            const __half2 hh = __floats2half2_rn(s0, s1);
            const float2 hf = __half22float2(hh);
            *reinterpret_cast<__half2*>(twd.hi + idx) = hh;
            *reinterpret_cast<__half2*>(twd.lo + idx) = __floats2half2_rn(s0 - hf.x, s1 - hf.y);
            m = fmax_nan(m, fmax_nan(fabsf(dv0), fabsf(dv1)));
          }
          db0 += dv0;
          db1 += dv1;
        }
      }
    }
  }
  if (twd.hi) twin_flush(twd, m, mul);
  if (i >= in) return;
  if (data)   // the node's pad rows (up to kNodeRowPad) carry zero deltas
    for (int r = n; r < (int)round_up(n, kNodeRowPad); ++r) {
      const size_t idx = (size_t)(r0 + r) * in + i;
      if (Dout) *reinterpret_cast<float2*>(Dout + idx) = make_float2(0.f, 0.f);
      if (twd.hi) {
        *reinterpret_cast<__half2*>(twd.hi + idx) = __floats2half2_rn(0.f, 0.f);
        *reinterpret_cast<__half2*>(twd.lo + idx) = __floats2half2_rn(0.f, 0.f);
      }
    }
  const float sw = *scale_w;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (o >= no) break;
    const long long q0 = quantise(g0[o], sw, lim, tail, tw);
    const long long q1 = quantise(g1[o], sw, lim, tail, tw);
    if (q0) atomicAdd(reinterpret_cast<unsigned long long*>(&Gw[(size_t)i * no + o]), (unsigned long long)q0);
    if (q1) atomicAdd(reinterpret_cast<unsigned long long*>(&Gw[(size_t)(i + 1) * no + o]), (unsigned long long)q1);
  }
  if (data) {
    const float sb = *scale_b;
    const long long q0 = quantise(db0, sb, lim, tail, tb);
    const long long q1 = quantise(db1, sb, lim, tail, tb);
    if (q0) atomicAdd(reinterpret_cast<unsigned long long*>(&Gb[i]), (unsigned long long)q0);
    if (q1) atomicAdd(reinterpret_cast<unsigned long long*>(&Gb[i + 1]), (unsigned long long)q1);
  }
}

// -------------------------------------------------------------------- SGD
// sync_gradients' rounding + x(1/B) (virtual_exec.cpp:169-174) and
// sgd_apply (model.cpp:364-374) fused: g = double(S) * 2^-s * (1/B);
// [v = mu*v + g]; w = w - lr*g in fp64 (no contraction), then refresh the
// fp32 copies W32 [in][out] and WT32 [out][in].  Skipped wholesale when the
// step hit a fixed-point overflow (the host lowers the scale and redoes it).
struct SgdArgs {
  double* w64;
  double* v64;          // momentum buffer or nullptr
  const long long* G;   // exact gradient sum (same layout as params)
  float* w32;
  float* wt32;          // transposed copy (weights only) or nullptr
  __half *w32h, *w32l;   // split-fp16 twins of w32 (or nullptr)
  Twin16 wtw;            // the weights' scale, max and range slot (kTailH16W)
  double* gout;         // optional mean-gradient export
  unsigned long long* gmax;  // max |g| of this tensor (bit pattern of a positive double)
  const unsigned long long* h16max;  // split-fp16 operand maxima of the step (global), h16n of them
  int h16n;
  const long long* tail;
  int ntail_flags;
  const StepParams* sp; // 2^-s per tensor, 1/B (virtual_exec.cpp:165), lr, mu
  float* wpad;          // whole-node kernel's padded weight image (or nullptr)
  int ldw;
  int tensor;
  int rows, cols;       // tensor shape (bias: rows = 1)
};

// Block-wide: did the step hit a non-finite value, a fixed-point overflow or
// a split-fp16 operand out of its range (kTailH16, or a global max|x| 2^sigma
// below kH16Under)?  One flag per thread, no serial chain of loads.
__device__ __forceinline__ bool block_poisoned(const long long* tail, int nflags,
                                               const StepParams* sp = nullptr,
                                               const unsigned long long* h16max = nullptr, int h16n = 0) {
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  const int nt = blockDim.x * blockDim.y;
  bool bad = false;
  if (t == 0) bad = tail[kTailNonfinite] != 0 || tail[kTailLossRange] != 0 || tail[kTailH16] != 0;
  for (int i = t; i < nflags; i += nt) bad |= tail[kTailOverflow + i] != 0;
  for (int i = t; i < h16n; i += nt) {
    const float m = __uint_as_float((uint32_t)h16max[i]);
    const float mul = sp->h16_mul[i];
    bad |= m > 0.f && m * mul < kH16Under && mul < 0x1p100f;
  }
  return __syncthreads_or(bad);
}

__device__ __forceinline__ double sgd_one(const SgdArgs& a, size_t k, float& w32) {
  const double g = __dmul_rn(__ll2double_rn(a.G[k]) * a.sp->inv_scale[a.tensor], a.sp->inv_b);
  double u = g;
  if (a.v64) {
    u = __dadd_rn(__dmul_rn(a.sp->mu, a.v64[k]), g);
    a.v64[k] = u;
  }
  const double w = __dsub_rn(a.w64[k], __dmul_rn(a.sp->lr, u));
  a.w64[k] = w;
  w32 = __double2float_rn(w);
  if (a.gout) a.gout[k] = g;
  return fabs(g);
}

// max |g| of the block into *dst: warp xor-max, then one atomic per block
// (per-warp atomics on one address serialise in L2 across thousands of blocks).
// Every thread of the block must call it.
__device__ __forceinline__ void block_max_to(unsigned long long* dst, double v) {
  __shared__ unsigned long long wmax[32];
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, b, s);
    b = o > b ? o : b;
  }
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  if ((t & 31) == 0) wmax[t >> 5] = b;
  __syncthreads();
  if (t == 0) {
    unsigned long long m = 0;
    for (int i = 0; i < nw; ++i) m = wmax[i] > m ? wmax[i] : m;
    if (m) atomicMax(dst, m);
  }
}

// Weight tensor: 64x32 (rows x cols) tiles, 32x8 threads, 8 elements per
// thread with all loads issued before the dependent math; transposed fp32 copy
// via smem.
// MOM: momentum buffer present (registers for v[] only then); TR: rows per tile.
template <bool MOM, int TR = 64>
__global__ void __launch_bounds__(256, MOM ? 2 : (TR <= 32 ? 4 : 3)) k_sgd_weight(SgdArgs a) {
  constexpr int TC = 32, PER = TR / 8;
  __shared__ float tile[TR][TC + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int c = c0 + tx;
  long long S[PER];
  double w[PER], v[MOM ? PER : 1];
#pragma unroll
  for (int k = 0; k < PER; ++k) {   // loads first: the poison check overlaps them
    const int r = r0 + ty + 8 * k;
    const bool ok = r < a.rows && c < a.cols;
    const size_t idx = (size_t)r * a.cols + c;
    S[k] = ok ? __ldg(a.G + idx) : 0;
    w[k] = ok ? a.w64[idx] : 0.0;
    if constexpr (MOM) v[k] = ok ? a.v64[idx] : 0.0;
  }
  if (block_poisoned(a.tail, a.ntail_flags, a.sp, a.h16max, a.h16n)) return;
  const double inv_scale = a.sp->inv_scale[a.tensor], inv_b = a.sp->inv_b;
  const double lr = a.sp->lr, mu = a.sp->mu;
  const float wmul = a.w32h ? *a.wtw.mul : 1.f;
  float wm = 0.f;
  double mx = 0.0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int r = r0 + ty + 8 * k;
    const bool ok = r < a.rows && c < a.cols;
    const double g = __dmul_rn(__ll2double_rn(S[k]) * inv_scale, inv_b);
    double u = g;
    if constexpr (MOM) u = __dadd_rn(__dmul_rn(mu, v[k]), g);
    const double wn = __dsub_rn(w[k], __dmul_rn(lr, u));
    const float w32 = __double2float_rn(wn);
    tile[ty + 8 * k][tx] = ok ? w32 : 0.f;
    if (ok) {
      const size_t idx = (size_t)r * a.cols + c;
      a.w64[idx] = wn;
      if constexpr (MOM) a.v64[idx] = u;
      if (a.w32) a.w32[idx] = w32;
      if (a.w32h) {
        put16(a.w32h, a.w32l, idx, w32, wmul);
        wm = fmax_nan(wm, fabsf(w32));
      }
      if (a.gout) a.gout[idx] = g;
      mx = fmax(mx, fabs(g));
    }
  }
  if (a.w32h) twin_flush(a.wtw, wm, wmul);
  block_max_to(a.gmax, mx);
  if (!a.wt32) return;
  __syncthreads();
  // transposed: WT[c][r], 32 columns x TR rows -> each warp row writes TR contiguous rows
#pragma unroll
  for (int k = 0; k < TC / 8; ++k) {
    const int cc = ty + 8 * k;
    const int col = c0 + cc;
    if (col >= a.cols) continue;
#pragma unroll
    for (int h = 0; h < TR / 32; ++h) {
      const int r = r0 + h * 32 + tx;
      if (r < a.rows) {
        const float v = tile[h * 32 + tx][cc];
        const size_t o = (size_t)col * a.rows + r;
        a.wt32[o] = v;
      }
    }
  }
}

// Weight tensor of a tcgen05 layer (only its split-fp16 twins are consumed,
// by the forward as an MN-major operand and by the bwd-data K-major: no
// transposed copy): 64x64 tiles, 32x8 threads, each thread two adjacent
// columns x 8 rows (16-B loads of S and w), the twins as half2.  Same
// per-element arithmetic as k_sgd_weight (same bits).  rows, cols even.
template <bool MOM>
__global__ void __launch_bounds__(256, 2) k_sgd_twins(SgdArgs a) {
  constexpr int TR = 64, TC = 64, PER = TR / 8;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int c = c0 + 2 * tx;
  longlong2 S[PER];
  double2 w[PER], v[MOM ? PER : 1];
#pragma unroll
  for (int k = 0; k < PER; ++k) {   // loads first: the poison check overlaps them
    const int r = r0 + ty + 8 * k;
    const bool ok = r < a.rows && c < a.cols;
    const size_t idx = (size_t)r * a.cols + c;
    S[k] = ok ? __ldg(reinterpret_cast<const longlong2*>(a.G + idx)) : make_longlong2(0, 0);
    w[k] = ok ? *reinterpret_cast<const double2*>(a.w64 + idx) : make_double2(0.0, 0.0);
    if constexpr (MOM) v[k] = ok ? *reinterpret_cast<const double2*>(a.v64 + idx) : make_double2(0.0, 0.0);
  }
  if (block_poisoned(a.tail, a.ntail_flags, a.sp, a.h16max, a.h16n)) return;
  const double inv_scale = a.sp->inv_scale[a.tensor], inv_b = a.sp->inv_b;
  const double lr = a.sp->lr, mu = a.sp->mu;
  const float wmul = *a.wtw.mul;
  float wm = 0.f;
  double mx = 0.0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int r = r0 + ty + 8 * k;
    const bool ok = r < a.rows && c < a.cols;
    const double g0 = __dmul_rn(__ll2double_rn(S[k].x) * inv_scale, inv_b);
    const double g1 = __dmul_rn(__ll2double_rn(S[k].y) * inv_scale, inv_b);
    double u0 = g0, u1 = g1;
    if constexpr (MOM) {
      u0 = __dadd_rn(__dmul_rn(mu, v[k].x), g0);
      u1 = __dadd_rn(__dmul_rn(mu, v[k].y), g1);
    }
    const double n0 = __dsub_rn(w[k].x, __dmul_rn(lr, u0));
    const double n1 = __dsub_rn(w[k].y, __dmul_rn(lr, u1));
    const float f0 = __double2float_rn(n0), f1 = __double2float_rn(n1);
    if (ok) {
      const size_t idx = (size_t)r * a.cols + c;
      *reinterpret_cast<double2*>(a.w64 + idx) = make_double2(n0, n1);
      if constexpr (MOM) *reinterpret_cast<double2*>(a.v64 + idx) = make_double2(u0, u1);
      const float s0 = f0 * wmul, s1 = f1 * wmul;
      const __half2 hh = __floats2half2_rn(s0, s1);
      const float2 hf = __half22float2(hh);
      *reinterpret_cast<__half2*>(a.w32h + idx) = hh;
      *reinterpret_cast<__half2*>(a.w32l + idx) = __floats2half2_rn(s0 - hf.x, s1 - hf.y);
      if (a.gout) *reinterpret_cast<double2*>(a.gout + idx) = make_double2(g0, g1);
      wm = fmax_nan(wm, fmax_nan(fabsf(f0), fabsf(f1)));
      mx = fmax(mx, fmax(fabs(g0), fabs(g1)));
    }
  }
  twin_flush(a.wtw, wm, wmul);
  block_max_to(a.gmax, mx);
}

// fp64 master -> fp32 working copies (set_params / resize seeding).
__global__ void k_refresh_weight(const double* __restrict__ w64, float* __restrict__ w32,
                                 float* __restrict__ wt32, int rows, int cols) {
  __shared__ float tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;
    float v = 0.f;
    if (r < rows && c < cols) {
      v = __double2float_rn(w64[(size_t)r * cols + c]);
      w32[(size_t)r * cols + c] = v;
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  if (!wt32) return;
  for (int k = ty; k < 32; k += 8) {
    const int c = c0 + k, r = r0 + tx;
    if (r < rows && c < cols) wt32[(size_t)c * rows + r] = tile[tx][k];
  }
}

__global__ void k_refresh_vec(const double* __restrict__ w64, float* __restrict__ w32, size_t n) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x)
    w32[k] = __double2float_rn(w64[k]);
}

}  // namespace vntb

namespace vntb {
// fp32 tensor -> its split-fp16 twins (an FFMA-produced operand of a tcgen05
// layer, the weights after set_params / a re-split).
__global__ void k_split16(const float* __restrict__ x, Twin16 t, size_t n) {
  const float mul = *t.mul;
  float m = 0.f;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x) {
    const float v = x[k];
    put16(t.hi, t.lo, k, v, mul);
    m = fmax_nan(m, fabsf(v));
  }
  twin_flush(t, m, mul);
}

// sync_gradients export: mean = double(S) * 2^-s * (1/B) (virtual_exec.cpp:162-166).
__global__ void k_mean_grad(const long long* __restrict__ G, double* __restrict__ out, size_t n,
                            double inv_scale, double inv_b) {
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x)
    out[k] = __dmul_rn(__ll2double_rn(G[k]) * inv_scale, inv_b);
}
}  // namespace vntb
