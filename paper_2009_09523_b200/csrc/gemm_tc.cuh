// tcgen05 / TMA tensor-core GEMMs for the wide dense layers (sm_100a).
//
// One kernel, three epilogues, all "TN" (both operands K-major in HBM):
//   forward    Z[r][n]  = X[l][r][:] . WT[l][n][:]        -> bias + f -> X[l+1], XT[l+1]
//   bwd-data   Dl[r][i] = D[l+1][r][:] . W[l][i][:]        -> * f'(X[l]) -> D[l], DT[l]
//   dW         per node k: g_k[i][o] = XT[l][i][cols_k] . DT[l+1][o][cols_k]
//              -> quantised to int64 and summed over the pass's nodes in
//                 registers, one store per tile (the virtual-node gradient
//                 accumulation fused into the GEMM epilogue).
// This file: the single-CTA kernel (128x128 dW tiles with VNT_TC_DW_PAIR=0,
// 128x256 fwd/bwd with VNT_TC_PAIR=0) and the shared pieces; the default
// CTA-pair kernels are in gemm_tc_pair.cuh.  Warp roles: w0 TMA producer (one
// lane), w1 MMA issuer (the whole warp runs the loop, one elected lane issues
// tcgen05.mma.kind::tf32; accumulators in TMEM), w2 TMEM allocator, w2..w9
// epilogue (tcgen05.ld, 32x32b).  Two operand formats (SPLIT): 1 = fp32
// tensors read by kind::tf32 (one pass), 3 = split-fp16 twins (x 2^sigma =
// hi + lo, kernels_simt.cuh) read by kind::f16 as hi*hi + hi*lo + lo*hi; a
// stage row is 128 B either way (32 tf32 or 64 fp16 K elements), so the
// tiling, swizzles and barriers are shared.  Smem operand tiles are 128B-swizzled
// K-major (TMA SWIZZLE_128B <-> UMMA SWIZZLE_128B descriptors); an mbarrier
// ring feeds the MMA warp; two TMEM accumulators let the epilogue of segment s
// overlap the MMAs of s+1.  Tiles are visited in groups of tile rows
// (tile_coords) so the resident tiles share operand panels in L2.
//
// Every output element is one K-chain over the same k-blocks in the same
// order whatever the row count or tile position, so results are independent
// of how many virtual nodes share a launch (the mapping-invariance contract).
#pragma once

#include <cuda.h>

#include "raster.cuh"

#include <algorithm>

namespace vntb {
namespace tc {

constexpr int BM = 128;

// Operand format of a SPLIT: element bytes, K elements per 128-B stage row
// (also the rows per stage and the features per 128-B group of the MN-major
// dW operands) and K per MMA instruction.
template <int SPLIT>
struct Fmt {
  static constexpr int EB = SPLIT == 3 ? 2 : 4;
  static constexpr int BKE = 128 / EB;
  static constexpr int KSTEP = 32 / EB;
  static constexpr uint32_t kGroupBytes = BKE * 128;   // an MN-major 128-B group of BKE rows
};
// w0 TMA, w1 MMA, w2..w9 epilogue (w2 also allocates TMEM): 320 threads leave
// the dW epilogue 204 registers for its 64 int64 accumulators (no spills).
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator
// (idle otherwise), warp 3 idle; warps 4..11 epilogue.  The first warpgroup
// gives registers to the epilogue warpgroups (setmaxnreg), which hold the
// promoted K-chunk sums (fwd / bwd) or the int64 node sums (dW) in registers.
constexpr int kEpiWarp0 = 4;
constexpr int kThreads = (kEpiWarp0 + 8) * 32;
constexpr int kRegsLow = 56, kRegsEpi = 224;   // 4 x 32 x 56 + 8 x 32 x 224 <= 64K

__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsLow));
}
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
}

enum : int { kTcFwd = 0, kTcBwd = 1, kTcDw = 2 };

// Diagnostics build only (-DVNT_TC_PROBE, scripts/tc_probe.py): cycles each
// role spends waiting on its barriers, per kernel kind (EPI + 3 * pair).
#ifdef VNT_TC_PROBE
__device__ unsigned long long g_tc_probe[6][16];   // 8..11: final-epilogue / promote cycles and counts; 12..15: finish phases
#define TC_PROBE_DECL long long _pw = 0, _pt = clock64()
#define TC_PROBE_WAIT(stmt)          \
  do {                               \
    const long long _t = clock64();  \
    stmt;                            \
    _pw += clock64() - _t;           \
  } while (0)
#define TC_PROBE_DONE(kind, slot)                                               \
  do {                                                                          \
    atomicAdd(&g_tc_probe[kind][slot], (unsigned long long)_pw);                \
    atomicAdd(&g_tc_probe[kind][slot + 1], (unsigned long long)(clock64() - _pt)); \
  } while (0)
#else
#define TC_PROBE_DECL
#define TC_PROBE_WAIT(stmt) stmt
#define TC_PROBE_DONE(kind, slot)
#endif

// fwd / bwd-data: 128x256 tiles (A 4 KB + B 8 KB of smem per 128-cycle MMA);
// dW: 128x128 (the int64 per-node accumulators live in registers).
template <int EPI, int SPLIT = 1>
struct TileCfg {
  static constexpr int BN = EPI == kTcDw ? 128 : 256;
  static constexpr int kBytesA = BM * 128;
  static constexpr int kBytesB = BN * 128;
  static constexpr int kStageBytes = (SPLIT == 3 ? 2 : 1) * (kBytesA + kBytesB);
  static constexpr int STAGES_MAX = EPI == kTcDw ? 6 : 4;
  static constexpr int STAGES = (192 * 1024 / kStageBytes) < STAGES_MAX ? (192 * 1024 / kStageBytes)
                                                                         : STAGES_MAX;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 + 256;
};

// Split-fp16: per k16 step hi*hi + hi*lo + lo*hi accumulate into one TMEM
// tile; the epilogue multiplies by 2^-(sigma_A + sigma_B) (exact).

struct EpiArgs {
  int M, N;
  // forward / bwd-data
  const float* bias;
  int act;
  float* out;
  int ldo;
  const float* Xprev;
  int ldx;
  // relu: f'(X) as a bit mask, [rows][ldm] words (bit j of word w = column
  // 32 w + j > 0) — written by the producing forward, read by the bwd-data
  // (the fp32 Xprev read in the final epilogue stalled the next tile's MMAs)
  uint32_t* mask_out;
  const uint32_t* mask_in;
  int ldm;
  // split-fp16 twins of out for the next tcgen05 consumer (tw.hi nullptr: none);
  // tma_out (CTA-pair fwd / bwd): 1 = the twins are the only output, 2 = the
  // plain fp32 out is (no twins); written by TMA stores from smem boxes
  Twin16 tw;
  int tma_out;
  // split-fp16 operands: 2^-sigma of A and B (nullptr: fp32 operands)
  const float* inv_a;
  const float* inv_b;
  // dW: per-node partial g -> rint(g * 2^s) (scale_p: 2^s of the tensor, read
  // per CTA from the step parameters), |g 2^s| < lim
  long long* G;
  int ldg;
  int first;
  const float* scale_p;
  float lim;
  int mn3;   // dW operand maps are 3-D (bit 0: A, bit 1: B), see make_map_mn3
  long long* tail;
  int tensor;
  // tile raster: groups of group_m tile rows, column-major inside a group, so
  // the tiles resident at once share A and B panels in L2 (0/1: row-major)
  int group_m;
  // fwd / bwd-data: K is accumulated in TMEM in chunks of kchunk columns
  // (multiple of Fmt::BKE; 0 = all of K at once) and the chunk sums are added in
  // fp32 registers in chunk order ("promotion").  tcgen05's TMEM accumulation
  // loses precision over long K chains (scripts/ubench_tf32_precision.cu:
  // split-fp16 at K = 4096 is 1.5e-5 of max|D| in one chain, 6.3e-7 in 128-column
  // chunks vs 2.3e-6 for an fp32 FMA chain).  The first chunk of a tile is
  // kfirst long: while it runs, the epilogue of the previous tile (its
  // output stores, bursty across all SMs) still holds the other buffer.
  int kchunk;
  int kfirst;
};

// K range [kb, kb + kl) of segment s: a virtual node's rows rounded up to
// kNodeRowPad (dW; pad rows carry zero deltas) or a K chunk (fwd/bwd).
__device__ __forceinline__ void seg_range(int s, int nseg, const int* seg_k0, const int* seg_rows, int K,
                                          int kchunk, int kfirst, int& kb, int& kl) {
  if (nseg > 0) {
    kb = seg_k0[s];
    kl = (int)round_up(seg_rows[s], kNodeRowPad);
  } else if (kchunk > 0) {
    kb = s == 0 ? 0 : kfirst + (s - 1) * kchunk;
    const int len = s == 0 ? kfirst : kchunk;
    kl = K - kb < len ? K - kb : len;
  } else {
    kb = 0;
    kl = K;
  }
}

__host__ __device__ inline int seg_count(int nseg, int K, int kchunk, int kfirst) {
  if (nseg > 0) return nseg;
  if (kchunk <= 0 || K <= kfirst) return 1;
  return 1 + (K - kfirst + kchunk - 1) / kchunk;
}




__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

// 3-D box {32 features, rows, feature groups} of an MN-major operand map
// (make_map_mn3): all 32-feature groups of a tile in one instruction.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"((uint64_t)tm), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"((uint64_t)tm), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: 8-row core groups
// 1024 B apart (SBO), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: kind::tf32, D fp32, A/B tf32, K-major (fwd /
// bwd-data) or MN-major (dW: bits 15/16; both operands are the row-major
// activations / deltas themselves, K = rows).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn = false, bool b_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// MN-major fp16 operand (split-fp16 dW): the plain 128-B swizzle, rows of
// 128 B (64 features), 8-row core groups 1024 B apart (SBO), the 64-feature
// groups of an operand tile Fmt<3>::kGroupBytes apart (LBO).  A k16 MMA step =
// 16 rows = 2048 B.
__device__ __forceinline__ uint64_t sdesc_sw128_mn16(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(Fmt<3>::kGroupBytes >> 4) << 16;   // LBO: next 64-feature group
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: next 8-row core group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, D fp32, A/B fp16.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool a_mn = false, bool b_mn = false) {
  return (1u << 4) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// MN-major tf32 operand: the only smem layout tcgen05 takes for it is the
// 128-B swizzle with 32-B atomicity (layout type SWIZZLE_128B_BASE32B; what a
// TMA box with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B lands in): rows of 128 B
// (32 features), 4-row atoms of 512 B (SBO), the 32-feature groups of an
// operand tile kMnGroupBytes apart (LBO).  A k8 MMA step = 8 rows = 1024 B.
constexpr uint32_t kMnGroupBytes = 32 * 32 * 4;   // one TMA box: 32 rows x 128 B
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(kMnGroupBytes >> 4) << 16;   // LBO: next 32-feature group
  d |= (uint64_t)(512 >> 4) << 32;             // SBO: next 4-row atom
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;                      // SWIZZLE_128B_BASE32B
  return d;
}

// The MMA role runs on a whole warp with warp-uniform operands; one elected
// lane issues (elect.sync inside the asm), so the compiler keeps descriptors in
// uniform registers instead of wrapping every tcgen05.mma in a per-lane loop.
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int SPLIT>
__device__ __forceinline__ void mma_op(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (SPLIT == 3) mma_f16(d, a, b, idesc, acc);
  else mma_tf32(d, a, b, idesc, acc);
}

template <int SPLIT>
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr) {
  if constexpr (SPLIT == 3) return sdesc_sw128_mn16(saddr);
  else return sdesc_sw128_mn(saddr);
}

template <int SPLIT>
__host__ __device__ constexpr uint32_t idesc_of(int M, int N, bool a_mn, bool b_mn) {
  return SPLIT == 3 ? idesc_f16(M, N, a_mn, b_mn) : idesc_tf32(M, N, a_mn, b_mn);
}

// Epilogue side of the split-fp16 outputs: this thread's max |x| (and the
// range flag) into the twins' words, once per kernel (see twin_flush).
__device__ __forceinline__ void tw_put(const Twin16& t, size_t o, float x, float mul, float& m) {
  put16(t.hi, t.lo, o, x, mul);
  m = fmax_nan(m, fabsf(x));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          su32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16-column variant for the dW epilogue: its 64 int64 accumulators per thread
// leave no room for a 32-register staging array under the 168-register cap
// (3 warps per SM sub-partition).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

// fwd / bwd epilogue, K-chunk promotion: fold a finished chunk of TMEM
// columns [col0, col0 + 32 NB) of this warp's lanes into the register sums
// (first: overwrite), or — on the last chunk — add the sums into TMEM
// (sum + last chunk) for the regular epilogue, which reads the total from
// there (holding the 128 sums through the epilogue would spill).  16 columns
// per TMEM access.
template <int NB>
__device__ __forceinline__ void promote_chunk(uint32_t taddr, float (&pacc)[NB][32], bool first,
                                              bool last) {
#pragma unroll
  for (int c = 0; c < 2 * NB; ++c) {
    float v[16];
    tmem_ld16(taddr + (uint32_t)(c * 16), v);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float& a = pacc[c >> 1][(c & 1) * 16 + j];
      if (last) v[j] = a + v[j];
      else a = first ? v[j] : a + v[j];
    }
    if (last) tmem_st16(taddr + (uint32_t)(c * 16), v);
  }
  if (last) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Persistent: CTA b processes tiles b, b + gridDim.x, ... (n fastest).  Per
// tile, nseg == 0 means one segment covering K; otherwise segment s covers K
// columns [seg_k0[s], seg_k0[s] + round_up(seg_rows[s], 32)) — one virtual node.
// Accumulator buffers alternate over the global (tile, segment) sequence, so the
// epilogue of one segment overlaps the MMAs of the next, across tiles too.
template <int EPI, int SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmAl, const __grid_constant__ CUtensorMap tmBl,
              int K, int nseg, const int* __restrict__ seg_k0, const int* __restrict__ seg_rows,
              EpiArgs ep) {
  using C = TileCfg<EPI, SPLIT>;
  using F = Fmt<SPLIT>;
  constexpr int BN = C::BN, STAGES = C::STAGES, BKE = F::BKE, GW = F::BKE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::kBytesA;
  uint8_t* sAl = sB + STAGES * C::kBytesB;                       // SPLIT == 3 only
  uint8_t* sBl = sAl + (SPLIT == 3 ? STAGES * C::kBytesA : 0);
  uint64_t* full = (uint64_t*)(smem + STAGES * C::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int segs = seg_count(nseg, K, EPI == kTcDw ? 0 : ep.kchunk, ep.kfirst);
  const int tiles_n = (int)ceil_div(ep.N, BN);
  const int tiles_m = (int)ceil_div(ep.M, BM);
  const int tiles = tiles_m * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
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
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int tm, tn;
        tile_coords(tile, tiles_m, tiles_n, ep.group_m, tm, tn);
        const int m0 = tm * BM, n0 = tn * BN;
        for (int s = 0; s < segs; ++s) {
          int kb, kl;
          seg_range(s, nseg, seg_k0, seg_rows, K, ep.kchunk, ep.kfirst, kb, kl);
          for (int k = 0; k < kl; k += BKE) {
            TC_PROBE_WAIT(mbar_wait(&empty[stage], phase ^ 1));
            mbar_expect_tx(&full[stage], C::kStageBytes);
            // A: MN-major for the dW (BKE rows of the row-major X per stage,
            // GW-feature 128-B groups F::kGroupBytes apart: one 3-D box when the
            // width allows, ep.mn3 bit 0, else a 2-D box per group), K-major
            // otherwise; B: MN-major for the dW (D) and the forward (W [in][out]
            // itself: no transposed copy), K-major for the bwd-data.
            if constexpr (EPI == kTcDw) {
              if (ep.mn3 & 1) {
                tma_load_3d(sA + stage * C::kBytesA, &tmA, &full[stage], 0, kb + k, m0 / GW);
                if (SPLIT == 3) tma_load_3d(sAl + stage * C::kBytesA, &tmAl, &full[stage], 0, kb + k, m0 / GW);
              } else {
#pragma unroll
                for (int g = 0; g < BM / GW; ++g) {
                  tma_load_2d(sA + stage * C::kBytesA + g * F::kGroupBytes, &tmA, &full[stage], m0 + GW * g, kb + k);
                  if (SPLIT == 3)
                    tma_load_2d(sAl + stage * C::kBytesA + g * F::kGroupBytes, &tmAl, &full[stage], m0 + GW * g,
                                kb + k);
                }
              }
            } else {
              tma_load_2d(sA + stage * C::kBytesA, &tmA, &full[stage], kb + k, m0);
              if (SPLIT == 3) tma_load_2d(sAl + stage * C::kBytesA, &tmAl, &full[stage], kb + k, m0);
            }
            if constexpr (EPI != kTcBwd) {
              if (ep.mn3 & 2) {
                tma_load_3d(sB + stage * C::kBytesB, &tmB, &full[stage], 0, kb + k, n0 / GW);
                if (SPLIT == 3) tma_load_3d(sBl + stage * C::kBytesB, &tmBl, &full[stage], 0, kb + k, n0 / GW);
              } else {
#pragma unroll
                for (int g = 0; g < BN / GW; ++g) {
                  tma_load_2d(sB + stage * C::kBytesB + g * F::kGroupBytes, &tmB, &full[stage], n0 + GW * g, kb + k);
                  if (SPLIT == 3)
                    tma_load_2d(sBl + stage * C::kBytesB + g * F::kGroupBytes, &tmBl, &full[stage], n0 + GW * g,
                                kb + k);
                }
              }
            } else {
              tma_load_2d(sB + stage * C::kBytesB, &tmB, &full[stage], kb + k, n0);
              if (SPLIT == 3) tma_load_2d(sBl + stage * C::kBytesB, &tmBl, &full[stage], kb + k, n0);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      TC_PROBE_DONE(EPI, 0);
    }
  } else if (warp == 1) {
    regs_dec();
    {
      constexpr bool a_mn = EPI == kTcDw, b_mn = EPI != kTcBwd;   // operand majors (producer above)
      constexpr uint32_t idesc = idesc_of<SPLIT>(BM, BN, a_mn, b_mn);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t it = 0;  // global (tile, segment) counter
      TC_PROBE_DECL;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        for (int s = 0; s < segs; ++s, ++it) {
          const int b = it & 1;
          TC_PROBE_WAIT(mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1));
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(b * BN);
          int kb, kl;
          seg_range(s, nseg, seg_k0, seg_rows, K, ep.kchunk, ep.kfirst, kb, kl);
          for (int k = 0; k < kl; k += BKE) {
#ifdef VNT_TC_PROBE
            { const long long _t = clock64(); mbar_wait(&full[stage], phase);
              atomicAdd(&g_tc_probe[EPI][6], (unsigned long long)(clock64() - _t)); }
#else
            mbar_wait(&full[stage], phase);
#endif
            tc_fence_after();
            const uint64_t ad = a_mn ? sdesc_mn<SPLIT>(su32(sA + stage * C::kBytesA)) : sdesc_sw128(su32(sA + stage * C::kBytesA));
            const uint64_t bd = b_mn ? sdesc_mn<SPLIT>(su32(sB + stage * C::kBytesB)) : sdesc_sw128(su32(sB + stage * C::kBytesB));
            const uint64_t ald = a_mn ? sdesc_mn<SPLIT>(su32(sAl + stage * C::kBytesA)) : sdesc_sw128(su32(sAl + stage * C::kBytesA));
            const uint64_t bld = b_mn ? sdesc_mn<SPLIT>(su32(sBl + stage * C::kBytesB)) : sdesc_sw128(su32(sBl + stage * C::kBytesB));
            // dW: a node's K-chain is its rows rounded up to kNodeRowPad (K
            // steps past that are rows of the next node: skipped); a K step
            // is KSTEP 128-B rows (MN-major), 32 B inside the row (K-major)
            constexpr int KS = F::KSTEP;
            const int ksteps = EPI == kTcDw ? min(BKE, kl - k) / KS : BKE / KS;
#pragma unroll
            for (int kk = 0; kk < BKE / KS; ++kk) {
              if (kk >= ksteps) break;
              const uint64_t oa = (uint64_t)(a_mn ? kk * KS * 8 : kk * 2);
              const uint64_t ob = (uint64_t)(b_mn ? kk * KS * 8 : kk * 2);
              mma_op<SPLIT>(d, ad + oa, bd + ob, idesc, (k > 0 || kk > 0) ? 1u : 0u);
              if (SPLIT == 3) {
                mma_op<SPLIT>(d, ad + oa, bld + ob, idesc, 1u);
                mma_op<SPLIT>(d, ald + oa, bd + ob, idesc, 1u);
              }
            }
            mma_commit(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tfull[b]);
        }
      }
      TC_PROBE_DONE(EPI, 2);
    }
  } else if (warp >= kEpiWarp0) {
    regs_inc();
    constexpr int COLS = BN / 2;          // columns per epilogue thread
    const int q = warp & 3;               // TMEM lane quarter this warp may access
    const int h = (warp - kEpiWarp0) >> 2;        // column half
    const int row = q * 32 + lane;        // tile row == TMEM lane
    // split-fp16 operands: TMEM holds the sums at 2^(sigma_A + sigma_B)
    const float unscale = ep.inv_a ? *ep.inv_a * *ep.inv_b : 1.f;
    const float dscale = EPI == kTcDw ? *ep.scale_p * unscale : 1.f;   // dW: 2^s of the tensor
    const float tmul = ep.tw.hi ? *ep.tw.mul : 1.f;
    float tmax = 0.f;   // max |x| of the twins written
    uint32_t it = 0;
    float amax = 0.f;   // NaN-propagating max |x|: NaN/inf partials end up in it
    TC_PROBE_DECL;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, ep.group_m, tm, tn);
      const int m0 = tm * BM, n0 = tn * BN;
      const int r = m0 + row;
      long long acc[EPI == kTcDw ? COLS : 1];
      if (EPI == kTcDw) {
#pragma unroll
        for (int j = 0; j < COLS; ++j) acc[j] = 0;
      }
      // fwd / bwd: 32 finished columns (tile column col) of this thread's row
      auto finish32 = [&](float (&v)[32], int col) {
        const int nb = n0 + col;
        if (r >= ep.M) return;
        if constexpr (SPLIT == 3) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= unscale;
        }
        if (EPI == kTcBwd && ep.mask_in) {
          // (a chunk past the width has no mask word: the row holds ldm words)
          const uint32_t m = nb < ep.N ? __ldg(ep.mask_in + (size_t)r * ep.ldm + nb / 32) : 0u;
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
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = nb + j;
            if (n < ep.N) {
              if (EPI == kTcFwd)
                v[j] = act_fwd(ep.act, v[j] + __ldg(ep.bias + n));
              else
                v[j] *= act_grad_from_out(ep.act, ep.Xprev[(size_t)r * ep.ldx + n]);
            }
          }
        }
        if (EPI == kTcFwd && ep.mask_out && nb < ep.N) {   // the row's ldm words cover [0, N) only
          uint32_t m = 0;
#pragma unroll
          for (int j = 0; j < 32; ++j) m |= (nb + j < ep.N && v[j] > 0.f ? 1u : 0u) << j;
          ep.mask_out[(size_t)r * ep.ldm + nb / 32] = m;
        }
        if (ep.out) {   // null: only the split-fp16 twins are consumed
          float* orow = ep.out + (size_t)r * ep.ldo + nb;
          if (nb + 32 <= ep.N) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(orow + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < ep.N) orow[j] = v[j];
          }
        }
        if (ep.tw.hi) {
          const size_t o = (size_t)r * ep.ldo + nb;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (nb + j < ep.N) tw_put(ep.tw, o + j, v[j], tmul, tmax);
        }
      };
      int s0 = 0;
      if constexpr (EPI != kTcDw) if (segs > 1) {
        // K-chunk promotion: chunks 0..segs-2 fold into registers (buffer
        // released at once); the sum is added into the last chunk's TMEM,
        // which the regular epilogue below reads (same it).
        float pacc[COLS / 32][32];
        const uint32_t lane_col = ((uint32_t)(q * 32) << 16) + (uint32_t)(h * COLS);
        for (int s = 0; s < segs; ++s, ++it) {
          const int b = it & 1;
          TC_PROBE_WAIT(mbar_wait(&tfull[b], (it >> 1) & 1));
          tc_fence_after();
          const bool last = s + 1 == segs;
          promote_chunk<COLS / 32>(tmem + lane_col + (uint32_t)(b * BN), pacc, s == 0, last);
          if (last) break;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
        s0 = segs - 1;
      }
      for (int s = s0; s < segs; ++s, ++it) {
        const int b = it & 1;
        TC_PROBE_WAIT(mbar_wait(&tfull[b], (it >> 1) & 1));
        tc_fence_after();
        if constexpr (EPI == kTcDw) {
          // Per-node quantisation.  The 2^s scale is already in
          // the DT operand (exact power-of-two scaling), so TMEM holds g*2^s:
          // track max|x| (NaN-propagating), convert, accumulate.
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
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
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
    if (warp == kEpiWarp0 && lane == 0) TC_PROBE_DONE(EPI, 4);
#endif
    if (EPI != kTcDw && ep.tw.hi) twin_flush(ep.tw, tmax, tmul);
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
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    VNT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw EngineError(9, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

// K-major operand [rows][K] (fp32, eb = 4, or fp16, eb = 2) with leading
// dimension ld (elements); box 128 B of K x box_rows, 128B swizzle, zero fill
// out of bounds.
inline CUtensorMap make_map(const void* base, uint64_t rows, uint64_t K, uint64_t ld,
                            uint32_t box_rows,
                            CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, int eb = 4) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {K, rows};
  const cuuint64_t strides[1] = {ld * (uint64_t)eb};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / eb), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 2, (void*)base, dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(9, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// Split-fp16 output twin [rows][cols] (leading dimension ld) for the
// epilogue's TMA stores: boxes of 32 columns (64 B) x 32 rows, 64-B swizzle.
inline CUtensorMap make_map_store16(const __half* base, uint64_t rows, uint64_t cols, uint64_t ld) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(9, "cuTensorMapEncodeTiled (store) failed: " + std::to_string(r));
  return m;
}

// Plain fp32 output [rows][cols] for the epilogue's TMA stores: boxes of 32
// columns (128 B) x 32 rows, 128-B swizzle.
inline CUtensorMap make_map_store32(const float* base, uint64_t rows, uint64_t cols, uint64_t ld) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(9, "cuTensorMapEncodeTiled (store32) failed: " + std::to_string(r));
  return m;
}

// MN-major dW operand [rows][F] (features contiguous, F a multiple of the
// group width gw = 128 B / eb) as a 3-D tensor {gw features, rows, F / gw
// groups}: a box {gw, gw rows, box_groups} puts the groups kGroupBytes apart
// in smem, the layout the MMA descriptor expects, in one TMA instruction.
// fp32: the 32-B-atom 128-B swizzle (tf32 MN-major); fp16: the plain one.
inline CUtensorMap make_map_mn3(const void* base, uint64_t rows, uint64_t F, uint64_t ld,
                                uint32_t box_groups, int eb = 4) {
  CUtensorMap m;
  const uint32_t gw = 128 / eb;
  const cuuint64_t dims[3] = {gw, rows, F / gw};
  const cuuint64_t strides[2] = {ld * (uint64_t)eb, (uint64_t)gw * eb};
  const cuuint32_t box[3] = {gw, gw, box_groups};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 3, (void*)base, dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 eb == 2 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw EngineError(9, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string(r));
  return m;
}

template <int EPI, int SPLIT>
inline void launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& al,
                        const CUtensorMap& bl, int M, int N, int K, int nseg, const int* seg_k0,
                        const int* seg_rows, const EpiArgs& ep, int sms, cudaStream_t s) {
  using C = TileCfg<EPI, SPLIT>;
  static bool attr = false;
  if (!attr) {
    VNT_CUDA(cudaFuncSetAttribute(k_gemm_tc<EPI, SPLIT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    attr = true;
  }
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, C::BN));
  const int grid = std::min(tiles, sms);
  k_gemm_tc<EPI, SPLIT><<<grid, kThreads, C::kSmemBytes, s>>>(a, b, al, bl, K, nseg, seg_k0,
                                                              seg_rows, ep);
  VNT_LAUNCH_CHECK();
}

}  // namespace tc
}  // namespace vntb

#include "gemm_tc_pair.cuh"

// ---------------------------------------------- engine glue (needs vnt_engine)
namespace {

// CTA pairs for forward / bwd-data (VNT_TC_PAIR=0 selects the single-CTA kernel).
bool tc_use_pair() {
  static const bool on = !(getenv("VNT_TC_PAIR") && getenv("VNT_TC_PAIR")[0] == '0');
  return on;
}

// dW on 256x128 CTA pairs (VNT_TC_DW_PAIR=0 selects the single-CTA 128x128
// kernel).  Per SM the pair reads half of B and writes half of B's
// stages into smem; with the whole-warp MMA issue it beats the single-CTA dW
// on cfg3 (profiles/r01_summary.md).
// 3-D TMA maps for the MN-major dW operands (VNT_TC_MN3=0: one 2-D box per group).
bool tc_mn3() {
  static const bool on = !(getenv("VNT_TC_MN3") && getenv("VNT_TC_MN3")[0] == '0');
  return on;
}

// TMA stores of the split-fp16 epilogue outputs (VNT_TC_TMA_OUT=0: per-lane stores).
bool tc_tma_out() {
  static const bool on = !(getenv("VNT_TC_TMA_OUT") && getenv("VNT_TC_TMA_OUT")[0] == '0');
  return on;
}

bool tc_dw_pair() {
  static const bool on = !(getenv("VNT_TC_DW_PAIR") && getenv("VNT_TC_DW_PAIR")[0] == '0');
  return on;
}

// Tile-raster group height (VNT_TC_GROUP_M, default 8; 1 = row-major order).
int tc_group_m() {
  static const int g = [] {
    const char* v = getenv("VNT_TC_GROUP_M");
    return v ? std::max(1, atoi(v)) : 8;
  }();
  return g;
}

// Split-fp16 operands need 16-byte row strides (widths % 8 == 0).
bool tc_layer_eligible(int mode, uint64_t in, uint64_t out) {
  if (mode == VNT_GEMM_FFMA) return false;
  const uint64_t a = mode == VNT_GEMM_TF32 ? 4 : 8;
  return in >= 64 && out >= 64 && in % a == 0 && out % a == 0;
}

void tc_init(vnt_engine*) {}
void tc_destroy(vnt_engine*) {}

// Operand maps: the fp32 tensor itself (1 pass, kind::tf32) or its split-fp16
// hi / lo twins (3 passes, kind::f16).
struct OpMaps {
  CUtensorMap hi, lo;
};

// mn_major: the dW operands (X / D rows as K, features contiguous) in the
// MN-major 128-B swizzle (32-B atoms for tf32); mn3_groups > 0: as 3-D maps
// loading that many 128-B feature groups per box (width % group == 0).
OpMaps op_maps(const vnt_engine* e, const float* full, const __half* hi, const __half* lo,
               uint64_t rows, uint64_t K, uint64_t ld, uint32_t box, bool mn_major = false,
               uint32_t mn3_groups = 0) {
  using namespace vntb::tc;
  const int eb = e->split ? 2 : 4;
  const CUtensorMapSwizzle swz =
      mn_major && !e->split ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  OpMaps m;
  if (mn3_groups) {
    m.hi = make_map_mn3(e->split ? (const void*)hi : (const void*)full, rows, K, ld, mn3_groups, eb);
    m.lo = e->split ? make_map_mn3(lo, rows, K, ld, mn3_groups, eb) : m.hi;
    return m;
  }
  if (e->split) {
    m.hi = make_map(hi, rows, K, ld, box, swz, eb);
    m.lo = make_map(lo, rows, K, ld, box, swz, eb);
  } else {
    m.hi = make_map(full, rows, K, ld, box, swz, eb);
    m.lo = m.hi;
  }
  return m;
}

// K elements per stage of the engine's operand format.
int tc_bke(const vnt_engine* e) { return e->split ? vntb::tc::Fmt<3>::BKE : vntb::tc::Fmt<1>::BKE; }

// K chunk of the fwd / bwd-data promotion (EpiArgs::kchunk): split-fp16 only —
// a 1-pass TF32 GEMM is bounded by its operand rounding, not the chain.
// VNT_TC_KCHUNK overrides (0 = one TMEM chain over all of K); rounded to the
// stage K.
int tc_kchunk(const vnt_engine* e) {
  static const int env = getenv("VNT_TC_KCHUNK") ? atoi(getenv("VNT_TC_KCHUNK")) : -1;
  if (env >= 0) return env == 0 ? 0 : (int)round_up((uint64_t)env, tc_bke(e));
  return e->split ? 256 : 0;
}
// First chunk of a tile (VNT_TC_KFIRST, default 512): it runs while the
// previous tile's epilogue still holds the other TMEM buffer.  Measured at
// cfg3 (scripts/sweep_kchunk.py, profiles/r02_summary.md).
int tc_kfirst(const vnt_engine* e) {
  static const int env = getenv("VNT_TC_KFIRST") ? atoi(getenv("VNT_TC_KFIRST")) : 512;
  return std::max(tc_bke(e), (int)round_up((uint64_t)std::max(env, 1), tc_bke(e)));
}

template <int EPI>
void tc_launch(vnt_engine* e, bool pair, const OpMaps& a, const OpMaps& b, int M, int N, int K,
               int nseg, const int* seg_k0, const int* seg_rows, vntb::tc::EpiArgs ep) {
  using namespace vntb::tc;
  // a pair fwd / bwd with one kind of output (the split-fp16 twins, or the
  // plain fp32 tensor): TMA stores
  OpMaps o = a;
  ep.tma_out = 0;
  if (EPI != kTcDw && pair && tc_tma_out()) {
    if (e->split && ep.tw.hi && !ep.out) {
      o.hi = make_map_store16(ep.tw.hi, (uint64_t)M, (uint64_t)N, (uint64_t)ep.ldo);
      o.lo = make_map_store16(ep.tw.lo, (uint64_t)M, (uint64_t)N, (uint64_t)ep.ldo);
      ep.tma_out = 1;
    } else if (ep.out && !ep.tw.hi && ep.ldo % 4 == 0) {
      o.hi = make_map_store32(ep.out, (uint64_t)M, (uint64_t)N, (uint64_t)ep.ldo);
      o.lo = o.hi;
      ep.tma_out = 2;
    }
  }
  // K <= 1024 (the 784-wide first layer) runs as one TMEM chain: its error
  // is within the promoted 4096 chains' (profiles/r02_tf32_precision_probe.txt)
  ep.kchunk = (EPI == kTcDw || K <= 1024) ? 0 : tc_kchunk(e);
  ep.kfirst = tc_kfirst(e);
  // The backward GEMMs share the GPU with the per-layer gradient reductions,
  // and with a sharded update the forward ones with the weight all-gathers:
  // they leave kCommSms SMs to the NCCL kernels (gemm_sms).
  const int sms = (EPI == kTcFwd && !e->shard) ? e->sm_count : e->gemm_sms;
  ep.group_m = tc_group_m();
  // CTA-pair kernels for all three GEMMs in both modes
  if (pair) {
    if (e->split)
      launch_gemm_pair<EPI, 3>(a.hi, b.hi, a.lo, b.lo, o.hi, o.lo, M, N, K, nseg, seg_k0, seg_rows, ep,
                               sms, e->stream);
    else
      launch_gemm_pair<EPI, 1>(a.hi, b.hi, a.lo, b.lo, o.hi, o.lo, M, N, K, nseg, seg_k0, seg_rows, ep,
                               sms, e->stream);
    e->launches++;
    return;
  }
  if (e->split)
    launch_gemm<EPI, 3>(a.hi, b.hi, a.lo, b.lo, M, N, K, nseg, seg_k0, seg_rows, ep, sms,
                        e->stream);
  else
    launch_gemm<EPI, 1>(a.hi, b.hi, a.lo, b.lo, M, N, K, nseg, seg_k0, seg_rows, ep, sms,
                        e->stream);
  e->launches++;
}

void tc_forward(vnt_engine* e, int l, int rows, bool last) {
  using namespace vntb::tc;
  const int K = (int)e->widths[l], N = (int)e->widths[l + 1];
  if (last) throw vntb::EngineError(1, "tcgen05 path does not produce logits");
  const bool pair = tc_use_pair();
  const uint32_t bn = pair ? PairCfg<kTcFwd>::BNH : TileCfg<kTcFwd>::BN;
  const uint64_t lda = l == 0 ? e->ld0 : (uint64_t)K;
  const OpMaps a = op_maps(e, e->X[l], e->Xh[l], e->Xl[l], rows, K, lda, BM);
  // B = W [in][out] itself as an MN-major operand (K = in rows, out features
  // contiguous): the forward needs no transposed copy of the weights
  const uint64_t wo = e->woff[l];
  const uint32_t gw = (uint32_t)tc_bke(e);
  const bool b3 = N % gw == 0 && tc_mn3();
  const OpMaps b = op_maps(e, e->w32 + wo, e->split ? e->w32h + wo : nullptr, e->split ? e->w32l + wo : nullptr,
                           (uint64_t)K, (uint64_t)N, (uint64_t)N, gw, true, b3 ? bn / gw : 0);
  EpiArgs ep{};
  ep.mn3 = b3 ? 2 : 0;
  ep.M = rows;
  ep.N = N;
  ep.bias = e->w32 + e->boff[l];
  ep.act = e->act;
  if (e->split) {
    ep.inv_a = h16_inv(e, h16_op_x(e, l));
    ep.inv_b = h16_inv(e, h16_op_w(e));
  }
  // Plain X only when a consumer reads it: a split-fp16 layer l+1 reads the
  // twins, and with relu its bwd-data takes f' from the mask bits; other
  // activations keep the plain X for f'.
  const bool twins = e->Xh[l + 1] != nullptr;
  ep.out = twins && e->Mk[l + 1] ? nullptr : e->X[l + 1];
  ep.ldo = N;
  // twins are allocated only when the consuming layer l+1 runs on tcgen05 in split-fp16
  if (twins) ep.tw = twin_of(e, e->Xh[l + 1], e->Xl[l + 1], h16_op_x(e, l + 1));
  ep.mask_out = e->Mk[l + 1];   // relu' bits for the tcgen05 bwd-data of layer l+1
  ep.ldm = e->Mk[l + 1] ? (int)mask_ld(e, l + 1) : 0;
  tc_launch<kTcFwd>(e, pair, a, b, rows, N, K, 0, nullptr, nullptr, ep);
}

void tc_backward_data(vnt_engine* e, int l, int rows) {
  using namespace vntb::tc;
  const int N = (int)e->widths[l], K = (int)e->widths[l + 1];
  const bool pair = tc_use_pair();
  const uint32_t bn = pair ? PairCfg<kTcBwd>::BNH : TileCfg<kTcBwd>::BN;
  const OpMaps a = op_maps(e, e->D[l + 1], e->Dh[l + 1], e->Dl[l + 1], rows, K, K, BM);
  const uint64_t wo = e->woff[l];
  const OpMaps b = op_maps(e, e->w32 + wo, e->split ? e->w32h + wo : nullptr,
                           e->split ? e->w32l + wo : nullptr, N, K, K, bn);
  EpiArgs ep{};
  ep.M = rows;
  ep.N = N;
  ep.act = e->act;
  if (e->split) {
    ep.inv_a = h16_inv(e, h16_op_d(e, l + 1));
    ep.inv_b = h16_inv(e, h16_op_w(e));
  }
  // k_db and a non-tcgen05 layer l-1 read the plain delta; with twins (a
  // split-fp16 layer l-1) k_db reads the twins instead
  ep.out = e->Dh[l] ? nullptr : e->D[l];
  ep.ldo = N;
  ep.Xprev = e->X[l];   // f' when there is no relu mask
  ep.ldx = N;
  if (e->Dh[l]) ep.tw = twin_of(e, e->Dh[l], e->Dl[l], h16_op_d(e, l));
  ep.mask_in = e->Mk[l];
  ep.ldm = e->Mk[l] ? (int)mask_ld(e, l) : 0;
  tc_launch<kTcBwd>(e, pair, a, b, rows, N, K, 0, nullptr, nullptr, ep);
}

// Per-node dW: A = X[l] (rows x in), B = D[l+1] (rows x out), both read as
// MN-major operands (boxes of one 128-B feature group x BKE rows), K = a
// node's rows.
void tc_weight_grad(vnt_engine* e, int l, const Pass& p, const int* row0, const int* nrows,
                    const float* scale_p, float lim, bool first, int tensor) {
  using namespace vntb::tc;
  const int M = (int)e->widths[l], N = (int)e->widths[l + 1];
  // CTA pairs (256x128, B's smem traffic per SM halved), see tc_dw_pair().
  const bool pair = tc_use_pair() && tc_dw_pair();
  const uint64_t rows = p.rows;
  const uint32_t gw = (uint32_t)tc_bke(e);   // features per 128-B group
  // 3-D maps (one TMA per operand and stage) where the width allows.
  // X[0] rows are padded to a multiple of the group (ld0, zero pad columns):
  // the 3-D box covers the last partial feature group from the pad
  const uint64_t lda = l == 0 ? e->ld0 : (uint64_t)M;
  const bool a3 = lda % gw == 0 && tc_mn3(), b3 = N % gw == 0 && tc_mn3();
  const uint32_t bgroups = (pair ? PairCfg<kTcDw, 3>::BNH : TileCfg<kTcDw>::BN) / gw;
  const OpMaps a = op_maps(e, e->X[l], e->Xh[l], e->Xl[l], rows, a3 ? lda : (uint64_t)M, lda, gw, true,
                           a3 ? BM / gw : 0);
  const OpMaps b = op_maps(e, e->D[l + 1], e->Dh[l + 1], e->Dl[l + 1], rows, N, N, gw, true,
                           b3 ? bgroups : 0);
  EpiArgs ep{};
  ep.mn3 = (a3 ? 1 : 0) | (b3 ? 2 : 0);
  ep.M = M;
  ep.N = N;
  ep.G = e->G + e->woff[l];
  ep.ldg = N;
  ep.first = first ? 1 : 0;
  ep.scale_p = scale_p;
  ep.lim = lim;
  ep.tail = e->tail;
  ep.tensor = tensor;
  if (e->split) {
    ep.inv_a = h16_inv(e, h16_op_x(e, l));
    ep.inv_b = h16_inv(e, h16_op_d(e, l + 1));
  }
  tc_launch<kTcDw>(e, pair, a, b, M, N, (int)rows, (int)p.nodes.size(), row0, nrows, ep);
}

}  // namespace
