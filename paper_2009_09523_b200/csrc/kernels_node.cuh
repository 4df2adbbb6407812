// Whole-node kernel for small all-FFMA models (the reference's smallest MLP,
// BASELINE configs 1/2: [784, 16, 10], micro-batch 16).
//
// At that size the layered kernels are launch-latency bound (~25 dependent
// launches per step for a few MFLOP).  Here one CTA runs one virtual node
// end to end out of shared memory — fp64 rows in, forward (model.cpp:270-287),
// loss and output delta (model.cpp:289-315), backward (model.cpp:317-338), and
// the node's dW/db sums — then quantises the per-node partials and adds them
// into the exact int64 gradient sum G, exactly like the layered
// path does.  The input statistics (model.cpp:101-121) depend on x only and
// run concurrently on the engine's side stream (k_vn_stats, k_stats_combine).
//
// Determinism: every value is a fixed-order fp32 chain over one row (forward,
// backward) or over the node's rows in ascending order (dW, db), so the
// result is a function of the node's rows only — independent of which device
// or pass runs the node.  The engine picks this path from the layer widths
// alone (never from rows or mapping), so every run of a model uses it.
#pragma once

#include <cooperative_groups.h>

namespace vntb {

constexpr int kNodeMaxLayers = 8;
constexpr int kNodeThreads = 512;
constexpr int kNodeOC = 16;       // outputs per strip / per forward task
constexpr int kNodeStrips = 2;    // dW strips per thread
constexpr int kNodeMaxStrips = kNodeThreads * kNodeStrips;

struct NodeArgs {
  const double* x;       // staged pass rows (row-major, fp64)
  const double* y;
  const int* row0;       // per node of the pass: first row, row count
  const int* nrows;
  const float* w32;      // fp32 parameters, reference layout (model.cpp:62-77)
  const float* wpad;     // weights as staged in shared memory: [K][node_ldw(N)] per layer
  int wpad_floats;       // multiple of 4
  int L;
  int w[kNodeMaxLayers + 1];
  int woff[kNodeMaxLayers], boff[kNodeMaxLayers];
  int nstrips;           // sum_l (w[l] + 1) * ceil(w[l+1] / kNodeOC)
  int act, loss;
  int rc;                // rows per shared-memory chunk
  const StepParams* sp;  // per-tensor 2^s
  float lim;
  long long* G;          // exact gradient sum (zeroed) + tail
  long long* tail;
  long long examples;    // the pass's rows, added to the tail by CTA 0
  int part_off;          // CL > 1: smem float offset of the partial-strip exchange area
};

// Shared-memory row strides: deltas padded to kNodeOC (aligned float4 strips),
// staged weights W[i][:] padded so ld/4 is odd (conflict-free float4 rows).
__host__ __device__ constexpr int node_ld(int w) { return (w + kNodeOC - 1) / kNodeOC * kNodeOC; }
__host__ __device__ constexpr int node_ldw(int n) { return (((n + 3) / 4) | 1) * 4; }

// Offset of layer l in the padded weight image (float4-aligned layers).
__host__ __device__ inline int node_wpad_offset(const int* w, int l) {
  int off = 0;
  for (int k = 0; k < l; ++k) off += (w[k] * node_ldw(w[k + 1]) + 3) & ~3;
  return off;
}

// w32 -> padded image of one layer (set_params / resize; the SGD keeps it current).
__global__ void k_node_pad(const float* __restrict__ W, float* __restrict__ wpad, int K, int N) {
  const int ldw = node_ldw(N);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < K * N; t += gridDim.x * blockDim.x) {
    const int i = t / N;
    wpad[i * ldw + (t - i * N)] = W[t];
  }
}

// Row loss + output delta of one row (k_loss's arithmetic), one warp.
__device__ __forceinline__ void node_row_loss(const float* z, const double* yr, int outw,
                                              int loss_kind, float* d, long long* tail,
                                              const StepParams* sp) {
  const int lane = threadIdx.x & 31;
  double loss = 0.0;
  if (loss_kind == 0) {
    for (int o = lane; o < outw; o += 32) {
      const double df = (double)z[o] - yr[o];
      loss += df * df;
      d[o] = (float)(2.0 * df / (double)outw);
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
      d[o] = (float)(exp(zm) / norm - yr[o]);
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, s);
  }
  long long q;
  if (lane == 0 && row_loss_q(loss, sp, tail, q))
    atomicAdd(reinterpret_cast<unsigned long long*>(&tail[kTailLoss]), (unsigned long long)q);
}

// dW/db strip s -> (layer l, input row i (== w[l]: the bias), first output o0).
// Strips run i fastest so a warp shares one D row segment (smem broadcast).
__device__ __forceinline__ void node_strip(const NodeArgs& a, int s, int& l, int& i, int& o0) {
  l = 0;
  for (;;) {
    const int nch = (a.w[l + 1] + kNodeOC - 1) / kNodeOC;
    const int cnt = (a.w[l] + 1) * nch;
    if (s < cnt || l + 1 == a.L) break;
    s -= cnt;
    ++l;
  }
  const int rowsl = a.w[l] + 1;
  o0 = (s / rowsl) * kNodeOC;
  i = s - (s / rowsl) * rowsl;
}

// CL > 1: a cluster of CL CTAs per node; CTA k runs rows [k n / CL, (k+1) n / CL)
// of the node (a split fixed by the node's row count), and the CTAs' dW/db
// strips are added in rank order over distributed shared memory before the
// quantisation — a fixed summation tree per node, so still a function of the
// node's rows only.
template <int CL>
__global__ void __launch_bounds__(kNodeThreads) k_node_step(NodeArgs a) {
  extern __shared__ float sm[];
  __shared__ int aoff[kNodeMaxLayers + 1], doff[kNodeMaxLayers + 1], wso[kNodeMaxLayers];
  const int node = blockIdx.x / CL;
  const int crank = (int)(blockIdx.x % CL);   // == %cluster_ctarank for 1-D clusters of CL
  const int node_rows = a.nrows[node];
  const int lo = crank * node_rows / CL, hi = (crank + 1) * node_rows / CL;
  const int r0 = a.row0[node] + lo, n = hi - lo;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int L = a.L, in = a.w[0], outw = a.w[L];
  if (tid == 0) {
    int off = 0;
    for (int l = 0; l <= L; ++l) {
      aoff[l] = off;
      off += a.rc * a.w[l];
    }
    off = (off + 3) & ~3;
    doff[0] = 0;
    for (int l = 1; l <= L; ++l) {
      doff[l] = off;
      off += a.rc * node_ld(a.w[l]);
    }
    off = (off + 3) & ~3;
    for (int l = 0; l < L; ++l) wso[l] = off + node_wpad_offset(a.w, l);
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.tail[kTailExamples]),
              (unsigned long long)a.examples);
  // per-strip quantisation scales, loaded before they are needed
  float qscale[kNodeStrips];
#pragma unroll
  for (int q = 0; q < kNodeStrips; ++q) {
    const int st = tid + q * nt;
    qscale[q] = 0.f;
    if (CL == 1 && st < a.nstrips) {
      int l, i, o0;
      node_strip(a, st, l, i, o0);
      qscale[q] = a.sp->scale[2 * l + (i == a.w[l] ? 1 : 0)];
    }
  }
  float g[kNodeStrips][kNodeOC];
#pragma unroll
  for (int q = 0; q < kNodeStrips; ++q)
#pragma unroll
    for (int j = 0; j < kNodeOC; ++j) g[q][j] = 0.f;

  for (int c0 = 0; c0 < n; c0 += a.rc) {
    const int rn = min(a.rc, n - c0);
    __syncthreads();
    {   // fp64 rows -> fp32 activations of layer 0; on the first chunk also the
        // padded weight image (written by the SGD).  Loads of both are issued
        // together, 8 x values and 4 weight float4s per thread in flight.
      float* A0 = sm + aoff[0];
      const double* xs = a.x + (size_t)(r0 + c0) * in;
      const int total = rn * in;
      const float4* wsrc = reinterpret_cast<const float4*>(a.wpad);
      float4* wdst = reinterpret_cast<float4*>(sm + wso[0]);
      const int n4 = c0 == 0 ? a.wpad_floats / 4 : 0;
      for (int t0 = tid, u0 = tid; t0 < total || u0 < n4; t0 += 8 * nt, u0 += 4 * nt) {
        double v[8];
        float4 wv[4];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int t = t0 + q * nt;
          v[q] = t < total ? __ldg(xs + t) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (u0 + q * nt < n4) wv[q] = __ldg(wsrc + u0 + q * nt);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int t = t0 + q * nt;
          if (t < total) A0[t] = __double2float_rn(v[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (u0 + q * nt < n4) wdst[u0 + q * nt] = wv[q];
      }
    }
    __syncthreads();
    // forward (model.cpp:280-286): one warp per (row, 16 outputs); lanes take
    // k = lane, lane+32, ... in ascending order, then a fixed xor tree, + bias.
    for (int l = 0; l < L; ++l) {
      const int K = a.w[l], N = a.w[l + 1], ldw = node_ldw(N);
      const int nch = (N + kNodeOC - 1) / kNodeOC;
      const float* Wl = sm + wso[l];
      const float* b = a.w32 + a.boff[l];
      const float* Ain = sm + aoff[l];
      float* Aout = sm + aoff[l + 1];
      const bool hidden = l < L - 1;
      for (int task = warp; task < rn * nch; task += nwarps) {
        const int r = task / nch, o0 = (task - (task / nch) * nch) * kNodeOC;
        const int on = min(kNodeOC, N - o0);
        const float* ar = Ain + r * K;
        float acc[kNodeOC];
#pragma unroll
        for (int j = 0; j < kNodeOC; ++j) acc[j] = 0.f;
#pragma unroll 2
        for (int k = lane; k < K; k += 32) {
          const float av = ar[k];
          const float4* wr = reinterpret_cast<const float4*>(Wl + k * ldw + o0);
#pragma unroll
          for (int j4 = 0; j4 < kNodeOC / 4; ++j4) {
            if (4 * j4 < on) {   // lanes beyond `on` accumulate padding, never stored
              const float4 wv = wr[j4];
              acc[4 * j4 + 0] = fmaf(av, wv.x, acc[4 * j4 + 0]);
              acc[4 * j4 + 1] = fmaf(av, wv.y, acc[4 * j4 + 1]);
              acc[4 * j4 + 2] = fmaf(av, wv.z, acc[4 * j4 + 2]);
              acc[4 * j4 + 3] = fmaf(av, wv.w, acc[4 * j4 + 3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kNodeOC; ++j) {
#pragma unroll
          for (int sft = 16; sft; sft >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], sft);
        }
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < kNodeOC; ++j)
          if (j == lane) v = acc[j];
        if (lane < on) {
          const float z = v + __ldg(b + o0 + lane);
          Aout[r * N + o0 + lane] = hidden ? act_fwd(a.act, z) : z;
        }
      }
      __syncthreads();
    }
    // loss + output delta, one warp per row
    for (int r = warp; r < rn; r += nwarps)
      node_row_loss(sm + aoff[L] + r * outw, a.y + (size_t)(r0 + c0 + r) * outw, outw, a.loss,
                    sm + doff[L] + r * node_ld(outw), a.tail, a.sp);
    __syncthreads();
    // backward (model.cpp:328-337): d[l][r][i] = (sum_o d[l+1][r][o] W[i][o]) f'(a[l][r][i]),
    // o ascending; lanes over i read W^T rows (coalesced).
    for (int l = L - 1; l >= 1; --l) {
      const int K = a.w[l], N = a.w[l + 1];
      const int ldn = node_ld(N), ldl = node_ld(K), ldw = node_ldw(N);
      const float* Wl = sm + wso[l];
      const float* Dn = sm + doff[l + 1];
      const float* Al = sm + aoff[l];
      float* Dl = sm + doff[l];
      const int nic = (K + 31) / 32;
      for (int task = warp; task < rn * nic; task += nwarps) {
        const int r = task / nic, i = (task - (task / nic) * nic) * 32 + lane;
        if (i < K) {
          const float* dr = Dn + r * ldn;
          const float* wr = Wl + i * ldw;
          float acc = 0.f;
          for (int o = 0; o < N; o += 4) {   // o ascending
            const float4 wv = *reinterpret_cast<const float4*>(wr + o);
            const float4 dv = *reinterpret_cast<const float4*>(dr + o);
            acc = fmaf(dv.x, wv.x, acc);
            if (o + 1 < N) acc = fmaf(dv.y, wv.y, acc);
            if (o + 2 < N) acc = fmaf(dv.z, wv.z, acc);
            if (o + 3 < N) acc = fmaf(dv.w, wv.w, acc);
          }
          Dl[r * ldl + i] = acc * act_grad_from_out(a.act, Al[r * K + i]);
        }
      }
      __syncthreads();
    }
    // this chunk's rows into the node's dW / db strips, rows ascending
#pragma unroll
    for (int q = 0; q < kNodeStrips; ++q) {
      const int st = tid + q * nt;
      if (st < a.nstrips) {
        int l, i, o0;
        node_strip(a, st, l, i, o0);
        const int K = a.w[l];
        const bool bias = i == K;
        const float* dc = sm + doff[l + 1] + o0;
        const int ldn = node_ld(a.w[l + 1]);
        const float* ac = sm + aoff[l] + (bias ? 0 : i);
        for (int r = 0; r < rn; ++r) {
          const float av = bias ? 1.f : ac[r * K];   // 1 * d is exact: db = sum_r d
          const float4* d4 = reinterpret_cast<const float4*>(dc + r * ldn);
#pragma unroll
          for (int j4 = 0; j4 < kNodeOC / 4; ++j4) {
            const float4 dv = d4[j4];
            g[q][4 * j4 + 0] = fmaf(av, dv.x, g[q][4 * j4 + 0]);
            g[q][4 * j4 + 1] = fmaf(av, dv.y, g[q][4 * j4 + 1]);
            g[q][4 * j4 + 2] = fmaf(av, dv.z, g[q][4 * j4 + 2]);
            g[q][4 * j4 + 3] = fmaf(av, dv.w, g[q][4 * j4 + 3]);
          }
        }
      }
    }
  }
  if constexpr (CL == 1) {
    // per-node quantisation into the exact sum (order-free int64 atomics)
#pragma unroll
    for (int q = 0; q < kNodeStrips; ++q) {
      const int st = tid + q * nt;
      if (st < a.nstrips) {
        int l, i, o0;
        node_strip(a, st, l, i, o0);
        const int K = a.w[l], N = a.w[l + 1];
        const bool bias = i == K;
        const int t = 2 * l + (bias ? 1 : 0);
        const float scale = qscale[q];
        long long* gp = a.G + (bias ? a.boff[l] : a.woff[l] + i * N) + o0;
#pragma unroll
        for (int j = 0; j < kNodeOC; ++j) {
          if (o0 + j < N) {
            const long long qv = quantise(g[q][j], scale, a.lim, a.tail, t);
            if (qv) atomicAdd(reinterpret_cast<unsigned long long*>(gp + j), (unsigned long long)qv);
          }
        }
      }
    }
  } else {
    // rank-order sum of the CTAs' partial strips over DSMEM, then quantise;
    // each CTA finishes a contiguous 1/CL of the strips
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    float* part = sm + a.part_off;
#pragma unroll
    for (int q = 0; q < kNodeStrips; ++q) {
      const int st = tid + q * nt;
      if (st < a.nstrips)
#pragma unroll
        for (int j = 0; j < kNodeOC; ++j) part[st * kNodeOC + j] = g[q][j];
    }
    cluster.sync();
    const float* parts[CL];
#pragma unroll
    for (int k = 0; k < CL; ++k) parts[k] = cluster.map_shared_rank(part, k);
    const int s0 = crank * a.nstrips / CL, s1 = (crank + 1) * a.nstrips / CL;
    for (int e = tid; e < (s1 - s0) * kNodeOC; e += nt) {
      const int st = s0 + e / kNodeOC, j = e % kNodeOC;
      int l, i, o0;
      node_strip(a, st, l, i, o0);
      const int K = a.w[l], N = a.w[l + 1];
      if (o0 + j >= N) continue;
      float v = parts[0][st * kNodeOC + j];
#pragma unroll
      for (int k = 1; k < CL; ++k) v += parts[k][st * kNodeOC + j];
      const bool bias = i == K;
      const int t = 2 * l + (bias ? 1 : 0);
      const long long qv = quantise(v, a.sp->scale[t], a.lim, a.tail, t);
      long long* gp = a.G + (bias ? a.boff[l] : a.woff[l] + i * N) + o0 + j;
      if (qv) atomicAdd(reinterpret_cast<unsigned long long*>(gp), (unsigned long long)qv);
    }
    cluster.sync();   // no CTA leaves while its partials may still be read
  }
}

// SGD of every tensor of a small model in one launch (blockIdx.y = tensor):
// sgd_one's arithmetic on each flat tensor (the layered path's bias vectors too), plus the padded weight image the
// whole-node kernel stages (no transposed copy is kept).
struct SgdMulti {
  SgdArgs t[2 * kNodeMaxLayers];
};

__global__ void __launch_bounds__(256) k_sgd_multi(const __grid_constant__ SgdMulti m) {
  const SgdArgs& a = m.t[blockIdx.y];
  if (block_poisoned(a.tail, a.ntail_flags, a.sp, a.h16max, a.h16n)) return;
  const size_t n = (size_t)a.rows * a.cols;
  double mx = 0.0;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x) {
    float w32;
    mx = fmax(mx, sgd_one(a, k, w32));
    a.w32[k] = w32;
    if (a.wpad) {
      const size_t i = k / a.cols;
      a.wpad[i * a.ldw + (k - i * a.cols)] = w32;
    }
  }
  block_max_to(a.gmax, mx);
}

}  // namespace vntb
