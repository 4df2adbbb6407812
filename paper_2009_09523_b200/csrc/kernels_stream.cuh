// Memory-bound kernels that stream their input through shared memory with
// bulk async copies (cp.async.bulk, the non-tensor TMA path) instead of
// register-held loads: the bytes in flight per SM are set by the smem ring,
// not by the register budget of the compute.
#pragma once

namespace vntb {

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          tc::su32(dst)),
      "l"((uint64_t)src), "r"(bytes), "r"(tc::su32(bar))
      : "memory");
}

// k_skinny_backward2 (kernels_simt.cuh) with the node's X[l] rows of the
// block's 256-feature slab streamed through a kSbStages-deep ring of 8-row
// stages (one elected thread issues a 1-KB bulk copy per row).  Same thread ↔
// feature-pair map and the same operation orders (dW chain over rows
// ascending, o ascending in the bwd-data dot product, db over rows ascending),
// so the results are bit-identical to k_skinny_backward2 / k_skinny_backward.
// The feature pair's arithmetic runs as packed FFMA2 (fma.rn.f32x2: per lane
// the same rounding as fmaf).  Requires in % 4 == 0 (16-B aligned rows and sizes).
constexpr int kSbStages = 4, kSbRows = 8, kSbSlab = 256;
// OUT bits: which results a launch produces (hoisted out of the row loop)
constexpr int kSbTwins = 1, kSbPlain = 2, kSbData = 4;

template <int NO, int ACT, int OUT>
__global__ void __launch_bounds__(128) k_skinny_backward_bulk(
    const float* __restrict__ X, const float* __restrict__ Dn, const float* __restrict__ W, int in, int no,
    const int* __restrict__ vn_row0, const int* __restrict__ vn_rows, float* __restrict__ Dout,
    Twin16 twd, const float* __restrict__ scale_w, long long* __restrict__ Gw, int tw,
    const float* __restrict__ scale_b, long long* __restrict__ Gb, int tb, float lim,
    long long* __restrict__ tail) {
  static_assert(NO % 4 == 0, "dn rows are read as float4");
  constexpr bool data = OUT & kSbData, twins = OUT & kSbTwins, plain = OUT & kSbPlain;
  __shared__ __align__(128) float xs[kSbStages][kSbRows][kSbSlab];
  __shared__ __align__(16) float dn[64][NO];
  __shared__ __align__(8) uint64_t bar[kSbStages];
  const int i0 = blockIdx.x * kSbSlab;
  const int tid = threadIdx.x;
  const int i = i0 + 2 * tid;
  const int v = blockIdx.y;
  const int r0 = vn_row0[v], n = vn_rows[v];
  const int nst = (n + kSbRows - 1) / kSbRows;
  const uint32_t row_bytes = (uint32_t)min(kSbSlab, in - i0) * 4u;
  const float mul = twins ? *twd.mul : 1.f;

  auto issue = [&](int j) {   // stage j: rows [8j, 8j + 8) of the node
    const int s = j % kSbStages;
    const int rows = min(kSbRows, n - j * kSbRows);
    tc::mbar_expect_tx(&bar[s], (uint32_t)rows * row_bytes);
    for (int r = 0; r < rows; ++r)
      bulk_g2s(&xs[s][r][0], X + (size_t)(r0 + j * kSbRows + r) * in + i0, row_bytes, &bar[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kSbStages; ++s) tc::mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < min(kSbStages, nst); ++j) issue(j);
  }

  float m = 0.f;
  // (feature i, feature i + 1) pairs: packed FFMA2, each lane the same fmaf
  float2 ww[NO], gg[NO];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const bool ok = data && i < in && o < no;
    ww[o].x = ok ? __ldg(W + (size_t)i * no + o) : 0.f;
    ww[o].y = ok ? __ldg(W + (size_t)(i + 1) * no + o) : 0.f;
    gg[o] = make_float2(0.f, 0.f);
  }
  float db0 = 0.f, db1 = 0.f;
  // one row: dW pair chains, the bwd-data dot product (o ascending), f', twins
  auto row = [&](const float2 a, const float* dr, size_t idx) {
    const float4* d4 = reinterpret_cast<const float4*>(dr);
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int o = 0; o < NO; o += 4) {
      const float4 d = d4[o / 4];
      const float2 dx = make_float2(d.x, d.x), dy = make_float2(d.y, d.y);
      const float2 dz = make_float2(d.z, d.z), dw = make_float2(d.w, d.w);
      gg[o] = __ffma2_rn(a, dx, gg[o]);
      gg[o + 1] = __ffma2_rn(a, dy, gg[o + 1]);
      gg[o + 2] = __ffma2_rn(a, dz, gg[o + 2]);
      gg[o + 3] = __ffma2_rn(a, dw, gg[o + 3]);
      if constexpr (data) {
        acc = __ffma2_rn(dx, ww[o], acc);
        acc = __ffma2_rn(dy, ww[o + 1], acc);
        acc = __ffma2_rn(dz, ww[o + 2], acc);
        acc = __ffma2_rn(dw, ww[o + 3], acc);
      }
    }
    if constexpr (data) {
      const float dv0 = acc.x * act_grad_from_out(ACT, a.x);
      const float dv1 = acc.y * act_grad_from_out(ACT, a.y);
      if constexpr (plain) *reinterpret_cast<float2*>(Dout + idx) = make_float2(dv0, dv1);
      if constexpr (twins) {
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
  };
  for (int c = 0; c < n; c += 64) {
    const int cn = min(64, n - c);
    __syncthreads();
    for (int k = tid; k < cn * NO; k += blockDim.x)
      dn[k / NO][k % NO] = (k % NO < no) ? Dn[(size_t)(r0 + c + k / NO) * no + k % NO] : 0.f;
    __syncthreads();
    for (int rr = 0; rr < cn; rr += kSbRows) {
      const int j = (c + rr) / kSbRows, s = j % kSbStages;
      tc::mbar_wait(&bar[s], (uint32_t)(j / kSbStages) & 1u);
      if (i < in) {
        const size_t base = (size_t)(r0 + c + rr) * in + i;
        if (rr + kSbRows <= cn) {
#pragma unroll
          for (int q = 0; q < kSbRows; ++q)
            row(*reinterpret_cast<const float2*>(&xs[s][q][2 * tid]), &dn[rr + q][0], base + (size_t)q * in);
        } else {
#pragma unroll 1
          for (int q = 0; q < cn - rr; ++q)
            row(*reinterpret_cast<const float2*>(&xs[s][q][2 * tid]), &dn[rr + q][0], base + (size_t)q * in);
        }
      }
      __syncthreads();   // stage s consumed by every thread: refill it
      if (tid == 0 && j + kSbStages < nst) issue(j + kSbStages);
    }
  }
  if constexpr (twins) twin_flush(twd, m, mul);
  if (i >= in) return;
  if constexpr (data)   // the node's pad rows (up to kNodeRowPad) carry zero deltas
    for (int r = n; r < (int)round_up(n, kNodeRowPad); ++r) {
      const size_t idx = (size_t)(r0 + r) * in + i;
      if constexpr (plain) *reinterpret_cast<float2*>(Dout + idx) = make_float2(0.f, 0.f);
      if constexpr (twins) {
        *reinterpret_cast<__half2*>(twd.hi + idx) = __floats2half2_rn(0.f, 0.f);
        *reinterpret_cast<__half2*>(twd.lo + idx) = __floats2half2_rn(0.f, 0.f);
      }
    }
  const float sw = *scale_w;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    if (o >= no) break;
    const long long q0 = quantise(gg[o].x, sw, lim, tail, tw);
    const long long q1 = quantise(gg[o].y, sw, lim, tail, tw);
    if (q0) atomicAdd(reinterpret_cast<unsigned long long*>(&Gw[(size_t)i * no + o]), (unsigned long long)q0);
    if (q1) atomicAdd(reinterpret_cast<unsigned long long*>(&Gw[(size_t)(i + 1) * no + o]), (unsigned long long)q1);
  }
  if constexpr (data) {
    const float sb = *scale_b;
    const long long q0 = quantise(db0, sb, lim, tail, tb);
    const long long q1 = quantise(db1, sb, lim, tail, tb);
    if (q0) atomicAdd(reinterpret_cast<unsigned long long*>(&Gb[i]), (unsigned long long)q0);
    if (q1) atomicAdd(reinterpret_cast<unsigned long long*>(&Gb[i + 1]), (unsigned long long)q1);
  }
}

// Host side: the activation and the output set as template arguments.
template <int NO, int ACT>
void launch_skinny_backward_bulk_act(dim3 grid, cudaStream_t s, int out, const float* X, const float* Dn,
                                     const float* W, int in, int no, const int* row0, const int* nrows,
                                     float* Dout, Twin16 twd, const float* scale_w, long long* Gw, int tw,
                                     const float* scale_b, long long* Gb, int tb, float lim, long long* tail) {
#define VNT_SB(O)                                                                                      \
  k_skinny_backward_bulk<NO, ACT, O><<<grid, 128, 0, s>>>(X, Dn, W, in, no, row0, nrows, Dout, twd, scale_w, \
                                                          Gw, tw, scale_b, Gb, tb, lim, tail)
  switch (out) {
    case 0: VNT_SB(0); break;
    case kSbData | kSbTwins: VNT_SB(kSbData | kSbTwins); break;
    case kSbData | kSbPlain: VNT_SB(kSbData | kSbPlain); break;
    default: VNT_SB(kSbData | kSbTwins | kSbPlain); break;
  }
#undef VNT_SB
}

template <int NO>
void launch_skinny_backward_bulk(cudaStream_t s, const float* X, const float* Dn, const float* W, int in, int no,
                                 int act, const int* row0, const int* nrows, int nn, float* Dout, Twin16 twd,
                                 const float* scale_w, long long* Gw, int tw, const float* scale_b, long long* Gb,
                                 int tb, float lim, long long* tail) {
  const dim3 grid((unsigned)((in + kSbSlab - 1) / kSbSlab), (unsigned)nn);
  const int out = Gb ? kSbData | (twd.hi ? kSbTwins : 0) | (Dout ? kSbPlain : 0) : 0;
  if (act == 0)
    launch_skinny_backward_bulk_act<NO, 0>(grid, s, out, X, Dn, W, in, no, row0, nrows, Dout, twd, scale_w, Gw,
                                           tw, scale_b, Gb, tb, lim, tail);
  else if (act == 1)
    launch_skinny_backward_bulk_act<NO, 1>(grid, s, out, X, Dn, W, in, no, row0, nrows, Dout, twd, scale_w, Gw,
                                           tw, scale_b, Gb, tb, lim, tail);
  else
    launch_skinny_backward_bulk_act<NO, 2>(grid, s, out, X, Dn, W, in, no, row0, nrows, Dout, twd, scale_w, Gw,
                                           tw, scale_b, Gb, tb, lim, tail);
}

}  // namespace vntb
