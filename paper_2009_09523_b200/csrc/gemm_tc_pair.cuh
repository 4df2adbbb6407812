// CTA-pair (cta_group::2) variant of the tcgen05 GEMM, the default for all
// three GEMMs.  A cluster of two CTAs (the two SMs of a TPC) computes a
// 256 x BN tile: CTA r owns A rows [m0 + 128 r, +128) and B rows
// [n0 + r BN/2, +BN/2) in its own smem; the leader (r = 0) issues
// tcgen05.mma.cta_group::2 on the pair's operands and each CTA receives its
// 128 accumulator rows in its own TMEM.  Per SM each CTA stages only half of
// B.  The fwd/bwd epilogue writes the split-fp16 twins of its
// output with TMA stores (a per-warp 32x32 box per twin staged in smem,
// 64-B swizzle), and a plain fp32 output, when one is needed, through a
// per-warp smem transpose tile so stores are 128 B rows (kEpiStageBytes).
#pragma once

namespace vntb {
namespace tc {

// fwd / bwd-data: 256x256 pair tiles; dW: 256x128 (each CTA keeps the int64
// per-node accumulators of its 128x128 half in registers, as the single-CTA dW).
template <int EPI, int SPLIT = 1>
struct PairCfg {
  static constexpr int BN = EPI == kTcDw ? 128 : 256;
  static constexpr int BNH = BN / 2;
  static constexpr int kBytesA = BM * 128;
  static constexpr int kBytesB = BNH * 128;
  static constexpr int kStageBytes = (SPLIT == 3 ? 2 : 1) * (kBytesA + kBytesB);
  static constexpr int STAGES = (192 * 1024 / kStageBytes) < 6 ? (192 * 1024 / kStageBytes) : 6;
  // TMEM accumulator buffers: fwd / bwd 2 x 256 columns; dW 4 x 128, so the
  // MMAs run up to three virtual nodes ahead of the per-node int64 epilogue
#ifndef VNT_DW_NBUF
#define VNT_DW_NBUF 4
#endif
  static constexpr int NBUF = EPI == kTcDw ? VNT_DW_NBUF : 2;
  static constexpr int kTmemCols = NBUF * BN;
  // fwd / bwd epilogue: a 32x33 fp32 transpose tile per epilogue warp
  static constexpr int kEpiStageBytes = EPI == kTcDw ? 0 : 8 * 32 * 33 * 4;
  // barriers in the first 256 B of a 1024-B block after the stages; the
  // epilogue staging (1024-B aligned for the swizzled TMA boxes) after it
  static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 + 1024 + kEpiStageBytes;
  static_assert(kSmemBytes <= 232448, "exceeds the opt-in shared memory per block");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

// Arrive on the leader CTA's copy of `bar` (same smem offset).  Used for the
// TMEM-empty handshake only: the TMEM reads are ordered by the caller's
// tcgen05.fence::before_thread_sync, so no cluster-scope release of generic
// memory is needed (a .release.cluster fence per virtual node stalls the dW
// epilogue on its own spill stores).
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n}" ::"r"(su32(bar))
      : "memory");
}

// TMA load into this CTA's smem; completion counted on the leader's barrier
// (peer bit 24 of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"((uint64_t)tm), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                                 int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"((uint64_t)tm), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void mma_f16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// TMA store of a 2-D box from this CTA's smem (bulk async group of the thread).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   (uint64_t)tm),
               "r"(su32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Whole-warp callers, one elected lane issues (see mma_tf32).
__device__ __forceinline__ void mma_tf32_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int SPLIT>
__device__ __forceinline__ void mma_op_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (SPLIT == 3) mma_f16_pair(d, a, b, idesc, acc);
  else mma_tf32_pair(d, a, b, idesc, acc);
}

__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}" ::"r"(su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __noinline__ float act_fwd_call(int act, float z) { return act_fwd(act, z); }

template <int EPI, int SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_tc_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmAl,
                   const __grid_constant__ CUtensorMap tmBl, const __grid_constant__ CUtensorMap tmOh,
                   const __grid_constant__ CUtensorMap tmOl, int K, int nseg,
                   const int* __restrict__ seg_k0, const int* __restrict__ seg_rows, EpiArgs ep) {
  using C = PairCfg<EPI, SPLIT>;
  using F = Fmt<SPLIT>;
  constexpr int BN = C::BN, BNH = C::BNH, STAGES = C::STAGES, PM = 2 * BM, BKE = F::BKE, GW = F::BKE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::kBytesA;
  uint8_t* sAl = sB + STAGES * C::kBytesB;
  uint8_t* sBl = sAl + (SPLIT == 3 ? STAGES * C::kBytesA : 0);
  uint64_t* full = (uint64_t*)(smem + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + C::NBUF;
  uint32_t* tmem_slot = (uint32_t*)(tempty + C::NBUF);
  float* stile = (float*)(smem + STAGES * C::kStageBytes + 1024);
  uint8_t* tstage = smem + STAGES * C::kStageBytes + 1024;   // TMA-store boxes (same region)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // dW: one K-chain per virtual node; fwd / bwd: K chunks (EpiArgs::kchunk)
  const int segs = seg_count(nseg, K, EPI == kTcDw ? 0 : ep.kchunk, ep.kfirst);
  const int tiles_n = (int)ceil_div(ep.N, BN);
  const int tiles_m = (int)ceil_div(ep.M, PM);
  const int tiles = tiles_m * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&tfull[b], 1);
      // dW: one arrival per CTA after its 8 epilogue warps meet on a named
      // barrier (per virtual node); fwd/bwd: every epilogue warp of both CTAs
      mbar_init(&tempty[b], EPI == kTcDw ? 2 : 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    regs_dec();
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      TC_PROBE_DECL;
      for (int tile = pair; tile < tiles; tile += npairs) {
        int tm, tn;
        tile_coords(tile, tiles_m, tiles_n, ep.group_m, tm, tn);
        const int m0 = tm * PM + (int)rank * BM;
        const int n0 = tn * BN + (int)rank * BNH;
        for (int sg = 0; sg < segs; ++sg) {
          int kb, kl;
          seg_range(sg, nseg, seg_k0, seg_rows, K, ep.kchunk, ep.kfirst, kb, kl);
          for (int k = 0; k < kl; k += BKE) {
            TC_PROBE_WAIT(mbar_wait(&empty[stage], phase ^ 1));
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
            // A: MN-major for the dW (BKE rows of the row-major X per stage,
            // GW-feature 128-B groups F::kGroupBytes apart: one 3-D box when the
            // width allows, ep.mn3 bit 0, else a 2-D box per group), K-major
            // otherwise; B: MN-major for the dW (D) and the forward (W [in][out]
            // itself: no transposed copy), K-major for the bwd-data.
            if constexpr (EPI == kTcDw) {
              if (ep.mn3 & 1) {
                tma_load_3d_pair(sA + stage * C::kBytesA, &tmA, &full[stage], 0, kb + k, m0 / GW);
                if (SPLIT == 3) tma_load_3d_pair(sAl + stage * C::kBytesA, &tmAl, &full[stage], 0, kb + k, m0 / GW);
              } else {
#pragma unroll
                for (int g = 0; g < BM / GW; ++g) {
                  tma_load_2d_pair(sA + stage * C::kBytesA + g * F::kGroupBytes, &tmA, &full[stage], m0 + GW * g, kb + k);
                  if (SPLIT == 3)
                    tma_load_2d_pair(sAl + stage * C::kBytesA + g * F::kGroupBytes, &tmAl, &full[stage], m0 + GW * g,
                                kb + k);
                }
              }
            } else {
              tma_load_2d_pair(sA + stage * C::kBytesA, &tmA, &full[stage], kb + k, m0);
              if (SPLIT == 3) tma_load_2d_pair(sAl + stage * C::kBytesA, &tmAl, &full[stage], kb + k, m0);
            }
            if constexpr (EPI != kTcBwd) {
              if (ep.mn3 & 2) {
                tma_load_3d_pair(sB + stage * C::kBytesB, &tmB, &full[stage], 0, kb + k, n0 / GW);
                if (SPLIT == 3) tma_load_3d_pair(sBl + stage * C::kBytesB, &tmBl, &full[stage], 0, kb + k, n0 / GW);
              } else {
#pragma unroll
                for (int g = 0; g < BNH / GW; ++g) {
                  tma_load_2d_pair(sB + stage * C::kBytesB + g * F::kGroupBytes, &tmB, &full[stage], n0 + GW * g, kb + k);
                  if (SPLIT == 3)
                    tma_load_2d_pair(sBl + stage * C::kBytesB + g * F::kGroupBytes, &tmBl, &full[stage], n0 + GW * g,
                                kb + k);
                }
              }
            } else {
              tma_load_2d_pair(sB + stage * C::kBytesB, &tmB, &full[stage], kb + k, n0);
              if (SPLIT == 3) tma_load_2d_pair(sBl + stage * C::kBytesB, &tmBl, &full[stage], kb + k, n0);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (rank == 0) TC_PROBE_DONE(EPI + 3, 0);
    }
  } else if (warp == 1) {
    regs_dec();
    if (rank == 0) {
      constexpr bool a_mn = EPI == kTcDw, b_mn = EPI != kTcBwd;   // operand majors (producer above)
      constexpr uint32_t idesc = idesc_of<SPLIT>(PM, BN, a_mn, b_mn);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t it = 0;
      TC_PROBE_DECL;
      for (int tile = pair; tile < tiles; tile += npairs)
      for (int sg = 0; sg < segs; ++sg, ++it) {
        const int b = (int)(it % C::NBUF);
        TC_PROBE_WAIT(mbar_wait_cluster(&tempty[b], ((it / C::NBUF) & 1) ^ 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        int kb, kl;
        seg_range(sg, nseg, seg_k0, seg_rows, K, ep.kchunk, ep.kfirst, kb, kl);
        for (int k = 0; k < kl; k += BKE) {
#ifdef VNT_TC_PROBE
          { const long long _t = clock64(); mbar_wait(&full[stage], phase);
            atomicAdd(&g_tc_probe[EPI + 3][6], (unsigned long long)(clock64() - _t)); }
#else
          mbar_wait(&full[stage], phase);
#endif
          tc_fence_after();
          const uint64_t ad = a_mn ? sdesc_mn<SPLIT>(su32(sA + stage * C::kBytesA)) : sdesc_sw128(su32(sA + stage * C::kBytesA));
          const uint64_t bd = b_mn ? sdesc_mn<SPLIT>(su32(sB + stage * C::kBytesB)) : sdesc_sw128(su32(sB + stage * C::kBytesB));
          const uint64_t ald = a_mn ? sdesc_mn<SPLIT>(su32(sAl + stage * C::kBytesA)) : sdesc_sw128(su32(sAl + stage * C::kBytesA));
          const uint64_t bld = b_mn ? sdesc_mn<SPLIT>(su32(sBl + stage * C::kBytesB)) : sdesc_sw128(su32(sBl + stage * C::kBytesB));
          constexpr int KS = F::KSTEP;
          // dW: node rows rounded to kNodeRowPad (K steps past them are the next node's rows)
          const int ksteps = EPI == kTcDw ? min(BKE, kl - k) / KS : BKE / KS;
#pragma unroll
          for (int kk = 0; kk < BKE / KS; ++kk) {
            if (kk >= ksteps) break;
            // a K step: KS 128-B rows (MN-major), 32 B inside the row (K-major)
            const uint64_t oa = (uint64_t)(a_mn ? kk * KS * 8 : kk * 2);
            const uint64_t ob = (uint64_t)(b_mn ? kk * KS * 8 : kk * 2);
            mma_op_pair<SPLIT>(d, ad + oa, bd + ob, idesc, (k > 0 || kk > 0) ? 1u : 0u);
            if (SPLIT == 3) {
              mma_op_pair<SPLIT>(d, ad + oa, bld + ob, idesc, 1u);
              mma_op_pair<SPLIT>(d, ald + oa, bd + ob, idesc, 1u);
            }
          }
          mma_commit_pair(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[b]);
      }
      TC_PROBE_DONE(EPI + 3, 2);
    }
  } else if (warp >= kEpiWarp0) {
    regs_inc();
    constexpr int COLS = BN / 2;
    const int q = warp & 3;
    const int h = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    const float unscale = ep.inv_a ? *ep.inv_a * *ep.inv_b : 1.f;   // split-fp16: 2^-(sigma_A + sigma_B)
    const float dscale = EPI == kTcDw ? *ep.scale_p * unscale : 1.f;   // dW: 2^s of the tensor
    const float tmul = ep.tw.hi ? *ep.tw.mul : 1.f;
    // TMA-stored twins: the epilogue works at the twins' scale 2^sigma_out
    // from the start (v = acc 2^-(sA+sB) 2^sigma_out, bias x 2^sigma_out):
    // power-of-two scaling commutes with the rounding, relu and the f' masks,
    // so the split sees the same bits (tmax is divided back at the end)
    const bool tscaled = SPLIT == 3 && ep.tma_out == 1;
    const float vscale = tscaled ? unscale * tmul : unscale;
    const float bscale = tscaled ? tmul : 1.f;
    float tmax = 0.f;   // max |x| of the twins written (x 2^sigma_out when tscaled)
    uint32_t it = 0;
    float amax = 0.f;   // NaN-propagating max |x|: NaN/inf partials end up in it
    TC_PROBE_DECL;
    for (int tile = pair; tile < tiles; tile += npairs) {
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, ep.group_m, tm, tn);
      const int m0 = tm * PM + (int)rank * BM, n0 = tn * BN;
      const int r = m0 + row;
      long long acc[EPI == kTcDw ? COLS : 1];
      if (EPI == kTcDw) {
#pragma unroll
        for (int j = 0; j < COLS; ++j) acc[j] = 0;
      }
      // bwd-data with a relu mask: this thread's 128 mask bits, loaded before
      // the K chunks so the final epilogue never waits on memory
      unsigned long long mk01 = 0, mk23 = 0;
      // fwd: this lane's bias of each 32-column chunk, loaded with the tile
      float bias_c[EPI == kTcFwd ? COLS / 32 : 1];
      if constexpr (EPI == kTcFwd) {
#pragma unroll
        for (int c = 0; c < COLS / 32; ++c) {
          const int n = n0 + h * COLS + 32 * c + lane;
          bias_c[c] = n < ep.N ? __ldg(ep.bias + n) * bscale : 0.f;
        }
      }
      if constexpr (EPI == kTcBwd) {
        // (a column half past the width has no mask words: the row holds ldm
        // = round_up(ceil(N / 32), 4) words)
        if (ep.mask_in && r < ep.M && n0 + h * COLS < ep.N) {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(ep.mask_in + (size_t)r * ep.ldm + (n0 + h * COLS) / 32));
          mk01 = (unsigned long long)w.x | ((unsigned long long)w.y << 32);
          mk23 = (unsigned long long)w.z | ((unsigned long long)w.w << 32);
        }
      }
      // fwd / bwd: 32 finished columns (tile column col) of this thread's row ->
      // bias + act (fwd) / f' (bwd), feature-major copies, row-major copies
      // through the per-warp smem transpose tile.
      auto finish32 = [&](float (&v)[32], int col) {
        const int nb = n0 + col;
#ifdef VNT_TC_PROBE
#ifndef VNT_PROBE_K
#define VNT_PROBE_K 0
#endif
        const bool _rec = lane == 0 && warp == kEpiWarp0 && rank == 0 && (VNT_PROBE_K == 0 || K == VNT_PROBE_K);
        long long _t0 = clock64();
#define FIN_MARK(slot)                                                          \
  do {                                                                          \
    const long long _t1 = clock64();                                            \
    if (_rec) atomicAdd(&g_tc_probe[EPI + 3][slot], (unsigned long long)(_t1 - _t0)); \
    _t0 = _t1;                                                                  \
  } while (0)
#else
#define FIN_MARK(slot)
#endif
        if constexpr (SPLIT == 3) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= vscale;
        }
        if constexpr (EPI == kTcFwd) {
          // bias: one coalesced load per warp, broadcast by shuffles
          // bias_c[] indexed by a select chain (a runtime index would move it to local memory)
          const int cc = (col - h * COLS) >> 5;
          float bl = bias_c[0];
#pragma unroll
          for (int c = 1; c < COLS / 32; ++c) bl = cc == c ? bias_c[c] : bl;
          // the activation switch outside the element loop: a per-element
          // act_fwd inlined 32 tanh bodies into the relu path (I-cache bound)
          if (ep.act == 0 && nb + 32 <= ep.N) {
            // relu, full chunk: the 32 biases as 8 broadcast 16-B loads (L1 hits)
            const float4* bp = reinterpret_cast<const float4*>(ep.bias + nb);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 b4 = __ldg(bp + j / 4);
              v[j] = fmaxf(fmaf(b4.x, bscale, v[j]), 0.f);   // relu (model.cpp:216)
              v[j + 1] = fmaxf(fmaf(b4.y, bscale, v[j + 1]), 0.f);
              v[j + 2] = fmaxf(fmaf(b4.z, bscale, v[j + 2]), 0.f);
              v[j + 3] = fmaxf(fmaf(b4.w, bscale, v[j + 3]), 0.f);
            }
          } else if (ep.act == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float bj = __shfl_sync(0xffffffffu, bl, j);
              if (nb + j < ep.N) v[j] = fmaxf(v[j] + bj, 0.f);
            }
          } else {
            // tanh / identity: out of line (a partially unrolled loop here would
            // move v[] to local memory for the whole epilogue)
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float bj = __shfl_sync(0xffffffffu, bl, j);
              if (nb + j < ep.N) v[j] = act_fwd_call(ep.act, v[j] + bj);
            }
          }
        }
        FIN_MARK(12);
        if constexpr (EPI == kTcFwd) {
          if (ep.mask_out && r < ep.M && nb < ep.N) {   // the row's ldm words cover [0, N) only
            uint32_t m = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) m |= (nb + j < ep.N && v[j] > 0.f ? 1u : 0u) << j;
            ep.mask_out[(size_t)r * ep.ldm + nb / 32] = m;
          }
        }
        FIN_MARK(13);
        if (r < ep.M) {
          if (EPI == kTcBwd && ep.mask_in) {
            const int c = (col - h * COLS) >> 5;
            const uint32_t m = (uint32_t)(((c & 2) ? mk23 : mk01) >> (32 * (c & 1)));
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= ((m >> j) & 1u) ? 1.f : 0.f;   // relu' (model.cpp:336)
          } else if (EPI == kTcBwd && nb + 32 <= ep.N) {
            const float4* xp = reinterpret_cast<const float4*>(ep.Xprev + (size_t)r * ep.ldx + nb);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 xv = __ldg(xp + j / 4);
              v[j] *= act_grad_from_out(ep.act, xv.x);
              v[j + 1] *= act_grad_from_out(ep.act, xv.y);
              v[j + 2] *= act_grad_from_out(ep.act, xv.z);
              v[j + 3] *= act_grad_from_out(ep.act, xv.w);
            }
          } else if (EPI == kTcBwd) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = nb + j;
              if (n < ep.N) v[j] *= act_grad_from_out(ep.act, ep.Xprev[(size_t)r * ep.ldx + n]);
            }
          }
        }
        if (ep.tma_out == 2) {
          // plain fp32 output only: this lane's row (128 B) into the warp's
          // 128-B-swizzled 32x32 box (chunk c of row r at c ^ (r & 7)), one
          // TMA store
          uint8_t* box = tstage + (warp - kEpiWarp0) * 4096;
          if (lane == 0) tma_store_wait_read();
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t off = (uint32_t)lane * 128 + (uint32_t)((c ^ (lane & 7)) * 16);
            *reinterpret_cast<float4*>(box + off) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmOh, box, nb, m0 + q * 32);
            tma_store_commit();
          }
          return;
        }
        if constexpr (SPLIT == 3) if (ep.tma_out == 1) {
          // split-fp16 twins only: this lane's row of the warp's 32x32 box,
          // hi and lo as 4 x 16 B each into the 64-B-swizzled staging boxes
          // (16-B chunk c of row r at chunk c ^ ((r >> 1) & 3): conflict-free),
          // then one TMA store per twin; rows / columns past the tensor are
          // clipped by the TMA unit
          uint8_t* box = tstage + (warp - kEpiWarp0) * 4096;
          if (lane == 0) tma_store_wait_read();   // the previous boxes were read out
          __syncwarp();
          FIN_MARK(14);
          // v is at the twins' scale already (tscaled); columns past N are
          // zero (zero-filled B rows, zero bias), rows past M are excluded
          if (r < ep.M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) tmax = fmax_nan(tmax, fabsf(v[j]));
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float x0 = v[8 * c + 2 * j], x1 = v[8 * c + 2 * j + 1];
              const __half2 hh = __floats2half2_rn(x0, x1);
              const float2 hf = __half22float2(hh);
              const __half2 ll = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
              h[j] = *reinterpret_cast<const uint32_t*>(&hh);
              l[j] = *reinterpret_cast<const uint32_t*>(&ll);
            }
            const uint32_t off = (uint32_t)lane * 64 + (uint32_t)((c ^ ((lane >> 1) & 3)) * 16);
            *reinterpret_cast<uint4*>(box + off) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(box + 2048 + off) = make_uint4(l[0], l[1], l[2], l[3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmOh, box, nb, m0 + q * 32);
            tma_store_2d(&tmOl, box + 2048, nb, m0 + q * 32);
            tma_store_commit();
          }
          FIN_MARK(15);
          return;
        }
        // row-major copies: transpose the warp's 32x32 block through smem so
        // every store writes 128 contiguous bytes of one row (a per-thread
        // float4 row store touches 32 lines per instruction)
        if (ep.out || ep.tw.hi) {
          float* st = stile + (warp - kEpiWarp0) * (32 * 33);
#pragma unroll
          for (int j = 0; j < 32; ++j) st[lane * 33 + j] = v[j];
          __syncwarp();
          const int n = nb + lane;
          const int rb = m0 + q * 32;
#pragma unroll 4
          for (int k = 0; k < 32; ++k) {
            const float x = st[k * 33 + lane];
            if (rb + k < ep.M && n < ep.N) {
              const size_t o = (size_t)(rb + k) * ep.ldo + n;
              if (ep.out) ep.out[o] = x;
              if (ep.tw.hi) tw_put(ep.tw, o, x, tmul, tmax);
            }
          }
          __syncwarp();
        }
      };
      int sg0 = 0;
      if constexpr (EPI != kTcDw) if (segs > 1) {
        // K-chunk promotion (EpiArgs::kchunk): chunks 0..segs-2 fold into
        // registers in chunk order (buffer released at once); the sum is
        // added into the last chunk's TMEM, which the epilogue below reads.
        float pacc[COLS / 32][32];
        const uint32_t lane_col = ((uint32_t)(q * 32) << 16) + (uint32_t)(h * COLS);
        for (int sg = 0; sg < segs; ++sg, ++it) {
          const int b = (int)(it % C::NBUF);
          TC_PROBE_WAIT(mbar_wait(&tfull[b], (it / C::NBUF) & 1));
          tc_fence_after();
          const bool last = sg + 1 == segs;
#ifdef VNT_TC_PROBE
          const long long _p0 = clock64();
#endif
          promote_chunk<COLS / 32>(tmem + lane_col + (uint32_t)(b * BN), pacc, sg == 0, last);
#ifdef VNT_TC_PROBE
          if (lane == 0 && warp == kEpiWarp0 && rank == 0) {
            atomicAdd(&g_tc_probe[EPI + 3][10], (unsigned long long)(clock64() - _p0));
            atomicAdd(&g_tc_probe[EPI + 3][11], 1ull);
          }
#endif
          if (last) break;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty[b]);
        }
        sg0 = segs - 1;
      }
      for (int sg = sg0; sg < segs; ++sg, ++it) {
      const int b = (int)(it % C::NBUF);
      TC_PROBE_WAIT(mbar_wait(&tfull[b], (it / C::NBUF) & 1));
      tc_fence_after();
#ifdef VNT_TC_PROBE
      const long long _f0 = clock64();
#endif
      if constexpr (EPI == kTcDw) {
        // per-node quantisation, as k_gemm_tc's dW epilogue
#pragma unroll
        for (int c = 0; c < COLS / 16; ++c) {
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + h * COLS + c * 16), v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float x = v[j] * dscale;   // exact: power of two
            amax = fmax_nan(amax, fabsf(x));
            acc[c * 16 + j] += __float2ll_rn(x);
          }
        }
      } else {
        // one 32-column chunk per iteration, not unrolled: the unrolled
        // epilogue overflowed the instruction cache (stall_no_inst at K = 784)
#pragma unroll 1
        for (int c = 0; c < COLS / 32; ++c) {
          float v[32];
          const int col = h * COLS + c * 32;
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN + col), v);
          finish32(v, col);
        }
      }
      tc_fence_before();
#ifdef VNT_TC_PROBE
      if (lane == 0 && warp == kEpiWarp0 && rank == 0 && (VNT_PROBE_K == 0 || K == VNT_PROBE_K)) {
        atomicAdd(&g_tc_probe[EPI + 3][8], (unsigned long long)(clock64() - _f0));
        atomicAdd(&g_tc_probe[EPI + 3][9], 1ull);
      }
#endif
      if (EPI == kTcDw) {
        asm volatile("bar.sync 1, 256;" ::: "memory");   // the 8 epilogue warps of this CTA
        if (warp == kEpiWarp0 && lane == 0) mbar_arrive_leader(&tempty[b]);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[b]);
      }
      }
      if (EPI == kTcDw && r < ep.M) {
        long long* g = ep.G + (size_t)r * ep.ldg + n0 + h * COLS;
        const int nvalid = ep.N - (n0 + h * COLS);
        if (nvalid >= COLS) {
#pragma unroll
          for (int j = 0; j < COLS; j += 2) {
            longlong2* gp = reinterpret_cast<longlong2*>(g + j);
            longlong2 o = ep.first ? make_longlong2(0, 0) : *gp;
            o.x += acc[j];
            o.y += acc[j + 1];
            *gp = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < COLS; ++j)
            if (j < nvalid) g[j] = ep.first ? acc[j] : g[j] + acc[j];
        }
      }
    }
#ifdef VNT_TC_PROBE
    if (warp == kEpiWarp0 && lane == 0 && rank == 0) TC_PROBE_DONE(EPI + 3, 4);
#endif
    if (EPI != kTcDw && ep.tw.hi) twin_flush(ep.tw, tscaled ? tmax * (1.f / tmul) : tmax, tmul);
    if (EPI != kTcDw && ep.tma_out && lane == 0) tma_store_wait_read();   // smem outlives the stores' reads
    if (EPI == kTcDw) {
      if (!(amax <= 3.402823466e38f))   // NaN or inf: some partial was non-finite
        atomicAdd(reinterpret_cast<unsigned long long*>(&ep.tail[kTailNonfinite]), 1ull);
      else if (!(amax < ep.lim))
        atomicAdd(reinterpret_cast<unsigned long long*>(&ep.tail[kTailOverflow + ep.tensor]), 1ull);
    }
  } else {
    regs_dec();   // warps 2, 3: the rest of the first warpgroup
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::kTmemCols)
                 : "memory");
  }
}

template <int EPI, int SPLIT>
inline void launch_gemm_pair(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& al,
                             const CUtensorMap& bl, const CUtensorMap& oh, const CUtensorMap& ol, int M,
                             int N, int K, int nseg, const int* seg_k0, const int* seg_rows,
                             const EpiArgs& ep, int sms, cudaStream_t s) {
  using C = PairCfg<EPI, SPLIT>;
  static bool attr = false;
  if (!attr) {
    VNT_CUDA(cudaFuncSetAttribute(k_gemm_tc_pair<EPI, SPLIT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    attr = true;
  }
  const int tiles = (int)(ceil_div(M, 2 * BM) * ceil_div(N, C::BN));
  const int pairs = std::max(1, std::min(tiles, sms / 2));
  k_gemm_tc_pair<EPI, SPLIT><<<2 * pairs, kThreads, C::kSmemBytes, s>>>(a, b, al, bl, oh, ol, K, nseg,
                                                                        seg_k0, seg_rows, ep);
  VNT_LAUNCH_CHECK();
}

}  // namespace tc
}  // namespace vntb
