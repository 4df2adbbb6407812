// B200 virtual-node training engine: the implementation behind the C-ABI in
// include/vnt_engine.h.  One process drives one GPU; the process hosts one or
// more logical devices (World workers, virtual_exec.hpp:100-114) and joins an
// NCCL group when world_size > 1.
//
// Step structure (train_step, virtual_exec.cpp:207-282):
//   passes of resident virtual nodes -> ingest + input stats -> forward layers
//   -> loss/delta -> backward (per-node dW/db quantised into the exact int64
//   sum, bwd-data; with an NCCL group each layer's slice is all-reduced as soon
//   as it is final, overlapped with the rest of the backward) -> fused rescale
//   + SGD -> control words (loss, examples, flags, max|g|) to mapped host memory.
// Small all-FFMA models replace the layered kernels of a pass with one
// whole-node kernel (kernels_node.cuh).  A single-pass step without an NCCL
// group is recorded once as a CUDA graph and replayed: every per-step value
// (scales, lr, batch pointers) reaches the kernels through the device
// StepParams block, so the launch sequence is static.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/vnt_engine.h"
#include "common.cuh"
#include "kernels_simt.cuh"
#include "kernels_node.cuh"
#include "kernels_shard.cuh"
#include "comm.cuh"

using namespace vntb;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

constexpr int kScaleTargetBits = 40;   // |sum| of the largest element ~ 2^40 after scaling
constexpr int kMaxRanks = 64;          // ranks of a sharded group (reduce-scatter overhang bound)
constexpr int kLimBits = 50;           // per-node partial bound for up to 2^12 partials
constexpr int kMaxPartialsLog2 = 21;   // beyond 2^21 partials the bound drops under the scale target
constexpr int kLossRescale = 16;       // loss quantum step on a loss-range redo
constexpr int kRescaleStep = 12;

struct PassNode {
  int node;          // global node id
  int dev;           // local device index
  uint64_t rows;     // node size
  uint64_t src_row;  // first row in the source batch
  uint64_t prow;     // first row in the pass (node rows padded to 8)
};

struct Pass {
  std::vector<PassNode> nodes;
  uint64_t rows = 0;       // pass rows, pad rows included
  uint64_t examples = 0;   // the nodes' rows (no padding)
  int* d_meta = nullptr;   // [valid(rows) | row0(n) | rows(n) | row0(n) | src_row(n)]
};

}  // namespace

struct vnt_engine {
  // model (ModelSpec, model.hpp:27-37; Layout, model.cpp:62-77)
  std::vector<uint64_t> widths;
  int L = 0;
  int act = 1, loss = 0;
  uint64_t P = 0;
  std::vector<uint64_t> woff, boff, wtoff;
  std::vector<int> tc_layer;   // 1: layer runs on tcgen05 tiles
  uint64_t ld0 = 0;             // row stride of X[0] (and twins): the input width, rounded
                                // up to 32 when layer 0 runs on tcgen05 (3-D TMA boxes of
                                // its MN-major dW operand); pad columns stay zero
  vnt_engine_options opt{};
  // Process groups: `pool` spans every process the job started (resize
  // migration runs over it); `comm` is the group that trains — the pool
  // itself, or a split of it after a resize left some processes idle — and
  // is null for a single process without a group.
  std::unique_ptr<vntb::CommGroup> pool;
  std::unique_ptr<vntb::CommGroup> active;   // owned split of the pool (when not the pool)
  vntb::CommGroup* comm = nullptr;
  // Per-layer gradient all-reduce overlapped with the rest of the backward:
  // layer l's slice of G is reduced on comm_stream as soon as its dW/db are
  // final, while the compute stream continues (VNT_COMM_OVERLAP=0 disables).
  bool comm_overlap = false;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> layer_ev;   // per layer: its dW/db done (compute stream)
  cudaEvent_t comm_ev = nullptr;       // comm_stream caught up
  int gemm_sms = 0;                    // CTAs the backward GEMMs may occupy
  std::vector<uint64_t> comm_log;      // (op, G offset, count) of every collective of a step
  // Sharded update (comm && layered path): layer l's gradient
  // slice is reduce-scattered into Gs, this rank updates its 1/G of the
  // parameters, and the new fp32 weights are all-gathered (deferred to the
  // next step's forward, layer by layer) and expanded into W's twins (or W / Wᵀ).
  bool shard = false;
  std::vector<uint64_t> sh_c, sh_lo, sh_hi, sh_soff, sh_aoff;   // per layer
  long long* Gs = nullptr;        // reduced chunks, sum_l c_l
  float* ag_send = nullptr;       // this rank's new fp32 weights, sum_l c_l
  float* ag_recv = nullptr;       // gathered slices, sum_l G c_l
  bool master_valid = true;       // w64 / v64 hold every element (not only this rank's)
  bool ag_pending = false;        // ag_send holds weights not yet gathered
  std::vector<char> ag_wait;      // per layer: gathered, not yet expanded
  std::vector<cudaEvent_t> ag_ev; // per layer: its all-gather done (comm stream)
  cudaEvent_t ag_fork = nullptr;
  long long* d_word = nullptr;    // 8 scratch words (count agreement)
  cudaStream_t stream = nullptr;
  int sm_count = 0;

  // replica state
  double* w64 = nullptr;
  double* v64 = nullptr;
  float* w32 = nullptr;
  float* wt32 = nullptr;
  long long* G = nullptr;   // P, a zero gap (reduce-scatter overhang), then the tail
  long long* tail = nullptr;   // G + tail_off: loss, examples, flags, then max|g| per tensor
  uint64_t tail_off = 0;
  size_t ntail = 0;
  unsigned long long* gmax = nullptr;
  double* gout = nullptr;
  std::vector<int> scales;
  bool scales_init = false;
  int lim_bits = kLimBits;             // |per-node partial| < 2^lim_bits (62 - log2 of the partial count)
  int loss_bits = kLossScaleBits;      // per-row loss quantum 2^-loss_bits (adapts on range flags)
  double loss_rows = 1;                // rows bound of the loss sum (power of two)
  uint64_t acc_partials = 0;           // per-node partials this process added in the round

  // pass buffers
  uint64_t cap_rows = 0, cap_vns = 0;
  double* xin = nullptr;   // = xbuf[cur]: the staged batch the kernels read
  double* yin = nullptr;
  double* xbuf[2] = {nullptr, nullptr};   // double-buffered input staging
  double* ybuf[2] = {nullptr, nullptr};
  int cur = 0;
  // next-step input prefetch (Trainer prefetch, runner.cpp:64-73, on the device)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t pf_event = nullptr;
  struct {
    const double* x = nullptr;
    const double* y = nullptr;
    int buf = -1;
    bool valid = false;
    std::vector<int64_t> layout;   // (node, dev, rows, src_row) of the staged rows
  } pf;
  // a second request waits until the in-flight one is consumed, then starts
  // right after the consuming step has launched its own work
  struct {
    const double* x = nullptr;
    const double* y = nullptr;
    uint64_t rows = 0;
    std::vector<uint64_t> sizes;
    std::vector<int32_t> devs;
    bool on_device = false;
    bool valid = false;
  } pf_next;
  std::vector<float*> X, D;
  // split-fp16 operand twins (x 2^sigma = hi + lo, kernels_simt.cuh), only when split.
  bool split = false;
  // whole-node kernel for small all-FFMA models (kernels_node.cuh)
  bool node_path = false;
  int node_rc_max = 0;
  int node_cl = 1;                     // CTAs per node (cluster size), fixed per model
  float* wpad = nullptr;               // padded weight image of k_node_step
  bool stats_backed = false;           // lineage stats backed up this round
  bool stats_join_pending = false;     // statistics branch not yet joined into the stream
  cudaStream_t aux_stream = nullptr;   // input-statistics branch beside k_node_step
  // VNT_HOST_PROFILE=1: host-side time per train_step phase (printed at destroy)
  bool host_prof = false;
  double host_t[8] = {};
  uint64_t host_n = 0;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  uint64_t tail_examples = 0;          // examples node kernels already added to the tail
  std::vector<__half*> Xh, Xl, Dh, Dl;
  // relu' of X[l] as bits [rows][mask_ld(l)] when both the producing forward
  // and the consuming bwd-data of X[l] run on tcgen05 (relu_mask(l))
  std::vector<uint32_t*> Mk;
  __half *w32h = nullptr, *w32l = nullptr;
  // split-fp16 operand scales: sigma per operand tensor (X[l] at l, D[l] at
  // L+1+l, all weights at 2L+2), chosen from the previous step's global max|x|
  // (h16max: one word per operand after gmax, max-reduced across ranks)
  std::vector<int> h16_sig;
  std::vector<int> h16_sig_step;   // the scales the last step ran with
  std::vector<std::pair<uint64_t, uint64_t>> last_rows;   // (pass row, rows) per node of the last pass
  unsigned long long* h16max = nullptr;
  unsigned long long* h_h16max = nullptr;
  float* logits = nullptr;
  double* vn_mean = nullptr;
  double* vn_m2 = nullptr;
  CombineStep* h_combine = nullptr;
  CombineStep* m_combine = nullptr;    // device view of the pinned h_combine
  size_t combine_cap = 0;
  long long* h_tail = nullptr;
  long long* m_tail = nullptr;         // device view of the pinned h_tail
  StepParams* m_sp = nullptr;          // device view of the pinned h_sp
  unsigned long long* h_gmax = nullptr;

  struct LDev {
    uint64_t capacity = 0;
    double count = 0;
    double* mean = nullptr;
    double* m2 = nullptr;
    double count_bak = 0;          // snapshot at round start (restored on rescale)
    double* mean_bak = nullptr;
    double* m2_bak = nullptr;
  };
  std::vector<LDev> devs;

  // plan cache (mapping -> passes with device-resident metadata)
  std::map<std::vector<int64_t>, std::vector<Pass>> plans;

  // accumulation state
  bool round_open = false;
  bool acc_started = false;
  uint64_t acc_examples = 0;
  bool synced = false;
  uint64_t total_nodes_hint = 0;

  // per-step kernel parameters (device copy read by kernels, pinned staging)
  StepParams* d_sp = nullptr;
  StepParams* h_sp = nullptr;
  // CUDA-graph replay of single-pass steps (VNT_GRAPHS=0 disables)
  struct GraphEntry {
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    uint32_t launches = 0;
    size_t prof_n = 0;
    std::vector<double> prof_flops;
  };
  bool graphs = true;
  bool timings_graphed = false;   // last step replayed a graph: only total_ms is timed
  std::map<std::vector<int64_t>, GraphEntry> graph_cache;
  // The mapping of the previous train_step and its graph entries by (cur,
  // stage-in-graph): a step with the same mapping skips rebuilding the node
  // list and the graph key (host time per step).  Cleared with the graphs.
  struct {
    std::vector<uint64_t> sizes;
    std::vector<int32_t> devs;
    uint64_t rows = 0;
    bool valid = false;
    GraphEntry* ge[2][2][2] = {};
  } memo;

  vnt_step_timings timings{};
  cudaEvent_t ev[6] = {};
  // Per-GEMM-launch device timing (CUDA events on the engine stream).
  bool profile = false;
  std::vector<cudaEvent_t> prof_ev;
  std::vector<double> prof_flops;
  size_t prof_n = 0;
  uint32_t launches = 0;
  std::vector<void*> scratch;
};

// X[l] gets a relu bit mask: written by a tcgen05 forward of layer l-1, read
// by the tcgen05 bwd-data of layer l.
bool relu_mask(const vnt_engine* e, int l) {
  return e->act == VNT_ACT_RELU && l >= 1 && l < e->L && e->tc_layer[l] && e->tc_layer[l - 1];
}
uint64_t mask_ld(const vnt_engine* e, int l) { return round_up(ceil_div(e->widths[l], 32), 4); }

// Split-fp16 operand ids (StepParams::h16_mul / h16_inv, h16max).
int h16_op_x(const vnt_engine*, int l) { return l; }
int h16_op_d(const vnt_engine* e, int l) { return e->L + 1 + l; }
int h16_op_w(const vnt_engine* e) { return 2 * e->L + 2; }
int h16_nops(const vnt_engine* e) { return 2 * e->L + 3; }
const float* h16_inv(vnt_engine* e, int op) { return &e->d_sp->h16_inv[op]; }
// Twins of operand `op` with its scale, max word and range flag (kTailH16:
// the step is redone; kTailH16W for the weight twins an update writes for
// the next step).
vntb::Twin16 twin_of(vnt_engine* e, __half* hi, __half* lo, int op, int flag = vntb::kTailH16) {
  vntb::Twin16 t{};
  t.hi = hi;
  t.lo = lo;
  t.mul = &e->d_sp->h16_mul[op];
  t.amax = e->h16max + op;
  t.flag = e->tail + flag;
  return t;
}

#include "gemm_tc.cuh"
#include "kernels_stream.cuh"

namespace {

void prof_begin(vnt_engine* e) {
  if (!e->profile) return;
  if (e->prof_n + 2 > e->prof_ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t ev;
      VNT_CUDA(cudaEventCreate(&ev));
      e->prof_ev.push_back(ev);
    }
  }
  VNT_CUDA(cudaEventRecord(e->prof_ev[e->prof_n], e->stream));  // prof_begin
}

void prof_end(vnt_engine* e, double flops) {
  if (!e->profile) return;
  VNT_CUDA(cudaEventRecord(e->prof_ev[e->prof_n + 1], e->stream));
  e->prof_n += 2;
  e->prof_flops.push_back(flops);
}

// After the step's final synchronisation: fold the GEMM launch times in.
void prof_collect(vnt_engine* e) {
  if (!e->profile) return;
  double ms_total = 0.0, fl = 0.0;
  for (size_t i = 0; i + 1 < e->prof_n; i += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e->prof_ev[i], e->prof_ev[i + 1]) != cudaSuccess) {
      (void)cudaGetLastError();   // timing unavailable: not an engine error
      ms = 0.f;
    }
    ms_total += ms;
  }
  for (double f : e->prof_flops) fl += f;
  e->timings.gemm_ms = (float)ms_total;
  e->timings.gemm_flops = fl;
  e->timings.gemm_launches = (uint32_t)(e->prof_n / 2);
  e->prof_n = 0;
  e->prof_flops.clear();
}

void* dalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  VNT_CUDA(cudaMalloc(&p, bytes));
  return p;
}

void bind(vnt_engine* e) { VNT_CUDA(cudaSetDevice(e->opt.cuda_device)); }

uint32_t ntensors(const vnt_engine* e) { return 2u * e->L; }

float pow2f(int s) { return std::ldexp(1.0f, s); }

const float* sp_scale(vnt_engine* e, int t) { return &e->d_sp->scale[t]; }

void drop_graphs(vnt_engine* e) {
  for (auto& kv : e->graph_cache)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  e->graph_cache.clear();
  e->memo.valid = false;
  for (auto& plane : e->memo.ge)
    for (auto& row : plane)
      for (auto& g : row) g = nullptr;
}

// Stage this step's kernel parameters (scales, 1/B, lr, momentum) for the device.
void fill_step_params(vnt_engine* e, double lr, double inv_b) {
  StepParams& h = *e->h_sp;
  for (uint32_t t = 0; t < ntensors(e); ++t) {
    h.scale[t] = pow2f(e->scales[t]);
    h.inv_scale[t] = std::ldexp(1.0, -e->scales[t]);
  }
  h.lr = lr;
  h.mu = e->opt.momentum;
  h.inv_b = inv_b;
  h.loss_scale = std::ldexp(1.0, e->loss_bits);
  h.loss_lim = std::ldexp(1.0, 62) / e->loss_rows;
  e->h16_sig_step = e->h16_sig;
  for (size_t op = 0; op < e->h16_sig.size(); ++op) {
    h.h16_mul[op] = std::ldexp(1.f, e->h16_sig[op]);
    h.h16_inv[op] = std::ldexp(1.f, -e->h16_sig[op]);
  }
}

// Pinned h_sp -> d_sp on the stream (a kernel reading mapped host memory, so it
// never waits behind an input prefetch on the copy engine); inside a captured
// step it re-reads h_sp at every replay.
void copy_step_params(vnt_engine* e) {
  static_assert(sizeof(StepParams) % 8 == 0, "StepParams words");
  k_copy_words<<<1, 256, 0, e->stream>>>(reinterpret_cast<const unsigned long long*>(e->m_sp),
                                         reinterpret_cast<unsigned long long*>(e->d_sp),
                                         (int)(sizeof(StepParams) / 8));
  VNT_LAUNCH_CHECK();
}

void upload_step_params(vnt_engine* e, double lr, double inv_b) {
  fill_step_params(e, lr, inv_b);
  copy_step_params(e);
}

int initial_scale(uint64_t batch) {
  // No gradient history: assume max |mean grad| ~ 1.
  return kScaleTargetBits - (int)std::ceil(std::log2((double)std::max<uint64_t>(batch, 1)));
}

void ensure_capacity(vnt_engine* e, uint64_t rows, uint64_t vns) {
  const int L = e->L;
  if (rows <= e->cap_rows && vns <= e->cap_vns) return;
  rows = std::max(rows, e->cap_rows);
  vns = std::max(vns, e->cap_vns);
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  if (e->copy_stream) VNT_CUDA(cudaStreamSynchronize(e->copy_stream));
  if (e->aux_stream) VNT_CUDA(cudaStreamSynchronize(e->aux_stream));
  e->stats_join_pending = false;
  e->pf.valid = false;
  drop_graphs(e);
  auto fre = [](auto*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  for (int b = 0; b < 2; ++b) {
    fre(e->xbuf[b]);
    fre(e->ybuf[b]);
  }
  e->xin = e->yin = nullptr;
  fre(e->logits);
  fre(e->vn_mean);
  fre(e->vn_m2);
  for (auto* v : {&e->X, &e->D})
    for (auto*& p : *v) fre(p);
  for (auto* v : {&e->Xh, &e->Xl, &e->Dh, &e->Dl})
    for (auto*& p : *v) fre(p);
  for (auto*& p : e->Mk) fre(p);
  const uint64_t in = e->widths[0], out = e->widths[L];
  for (int b = 0; b < 2; ++b) {
    e->xbuf[b] = (double*)dalloc(rows * in * sizeof(double));
    e->ybuf[b] = (double*)dalloc(rows * out * sizeof(double));
  }
  e->xin = e->xbuf[e->cur];
  e->yin = e->ybuf[e->cur];
  e->logits = (float*)dalloc(rows * out * sizeof(float));
  e->vn_mean = (double*)dalloc(vns * in * sizeof(double));
  e->vn_m2 = (double*)dalloc(vns * in * sizeof(double));
  for (auto* v : {&e->X, &e->D}) v->assign(L + 1, nullptr);
  for (auto* v : {&e->Xh, &e->Xl, &e->Dh, &e->Dl}) v->assign(L + 1, nullptr);
  e->Mk.assign(L + 1, nullptr);
  for (int l = 1; l < L; ++l)
    if (relu_mask(e, l)) e->Mk[l] = (uint32_t*)dalloc(rows * mask_ld(e, l) * sizeof(uint32_t));
  for (int l = 0; l <= L; ++l) {
    const uint64_t w = e->widths[l];
    const uint64_t wx = l == 0 ? e->ld0 : w;   // X row stride
    if (l < L) {
      e->X[l] = (float*)dalloc(rows * wx * sizeof(float));
      if (wx != w) VNT_CUDA(cudaMemset(e->X[l], 0, rows * wx * sizeof(float)));
    }
    if (l > 0) e->D[l] = (float*)dalloc(rows * w * sizeof(float));
    if (e->split) {
      if (l < L && e->tc_layer[l]) {   // operands of layer l: X[l] (fwd; dW, MN-major)
        e->Xh[l] = (__half*)dalloc(rows * wx * sizeof(__half));
        e->Xl[l] = (__half*)dalloc(rows * wx * sizeof(__half));
        if (wx != w) {
          VNT_CUDA(cudaMemset(e->Xh[l], 0, rows * wx * sizeof(__half)));
          VNT_CUDA(cudaMemset(e->Xl[l], 0, rows * wx * sizeof(__half)));
        }
      }
      if (l > 0 && e->tc_layer[l - 1]) {   // D[l] (bwd-data of l-1; dW of l-1, MN-major)
        e->Dh[l] = (__half*)dalloc(rows * w * sizeof(__half));
        e->Dl[l] = (__half*)dalloc(rows * w * sizeof(__half));
      }
    }
  }
  e->cap_rows = rows;
  e->cap_vns = vns;
}

void ensure_combine(vnt_engine* e, size_t n) {
  if (n <= e->combine_cap) return;
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  drop_graphs(e);
  if (e->h_combine) cudaFreeHost(e->h_combine);
  n = std::max<size_t>(n, 64);
  VNT_CUDA(cudaMallocHost(&e->h_combine, n * sizeof(CombineStep)));
  VNT_CUDA(cudaHostGetDevicePointer((void**)&e->m_combine, e->h_combine, 0));
  e->combine_cap = n;
}

// Device bytes per pass row (the buffers ensure_capacity allocates).
uint64_t pass_row_bytes(const vnt_engine* e) {
  const uint64_t in = e->widths[0], out = e->widths[e->L];
  uint64_t b = 2 * (in + out) * sizeof(double) + out * sizeof(float);   // staging x2, logits
  for (int l = 0; l <= e->L; ++l) {
    const uint64_t w = e->widths[l] * sizeof(float);
    const uint64_t wx = (l == 0 ? e->ld0 : e->widths[l]) * sizeof(float);
    if (l < e->L) b += wx * (e->split && e->tc_layer[l] ? 2 : 1);           // X (+ fp16 twins)
    if (l > 0) b += w * (e->split && e->tc_layer[l - 1] ? 2 : 1);           // D (+ fp16 twins)
    if (relu_mask(e, l)) b += mask_ld(e, l) * sizeof(uint32_t);
  }
  return b;
}

// Rows of one pass when the caller set no resident_rows: as many as 85 % of
// the free HBM holds (counting the pass buffers already allocated).  A node's
// own size is bounded by its device's memory_capacity (CapacityError), as in
// the reference's device_step; how many nodes are resident together is the
// B200's memory, not the model's.
uint64_t hbm_row_budget(vnt_engine* e) {
  size_t free_b = 0, total_b = 0;
  VNT_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t row = pass_row_bytes(e);
  const double usable = 0.85 * ((double)free_b + (double)(e->cap_rows * row));
  return std::max<uint64_t>(1, (uint64_t)(usable / (double)row));
}

// Group local nodes (ascending id) into passes that fit the resident-row budget
// (vnt_engine_options::resident_rows, else hbm_row_budget).
std::vector<Pass>& plan_for(vnt_engine* e, const std::vector<PassNode>& local) {
  std::vector<int64_t> key;
  key.reserve(local.size() * 4 + 1);
  key.push_back((int64_t)e->opt.resident_rows);
  for (const auto& n : local) {
    key.push_back(n.node);
    key.push_back(n.dev);
    key.push_back((int64_t)n.rows);
    key.push_back((int64_t)n.src_row);
  }
  auto it = e->plans.find(key);
  if (it != e->plans.end()) return it->second;
  std::vector<Pass> passes;
  const uint64_t budget = e->opt.resident_rows ? e->opt.resident_rows : hbm_row_budget(e);
  Pass cur;
  for (const auto& n : local) {
    if (!cur.nodes.empty() && cur.examples + n.rows > budget) {
      passes.push_back(cur);
      cur = Pass{};
    }
    PassNode pn = n;
    pn.prow = cur.rows;
    cur.rows += round_up(n.rows, kNodeRowPad);   // a node's dW K-chain runs in whole MMA K steps
    cur.examples += n.rows;
    cur.nodes.push_back(pn);
  }
  if (!cur.nodes.empty()) passes.push_back(cur);
  for (auto& p : passes) {
    const size_t nn = p.nodes.size();
    std::vector<int> meta(p.rows + 4 * nn, 0);
    for (size_t k = 0; k < nn; ++k) {
      const auto& pn = p.nodes[k];
      for (uint64_t r = 0; r < pn.rows; ++r) meta[pn.prow + r] = 1;   // pad rows stay 0
      meta[p.rows + k] = (int)pn.prow;
      meta[p.rows + nn + k] = (int)pn.rows;
      meta[p.rows + 2 * nn + k] = (int)pn.prow;
      meta[p.rows + 3 * nn + k] = (int)pn.src_row;
    }
    p.d_meta = (int*)dalloc(meta.size() * sizeof(int));
    VNT_CUDA(cudaMemcpy(p.d_meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  return e->plans.emplace(key, std::move(passes)).first->second;
}

// Tail and the per-tensor max|g| words sit back to back after G: one memset, one readback.
// Words zeroed per step after G: tail, per-tensor max|g|, split-fp16 maxima.
size_t tail_words(const vnt_engine* e) { return e->ntail + ntensors(e) + (size_t)h16_nops(e); }

void tail_reset(vnt_engine* e) {
  VNT_CUDA(cudaMemsetAsync(e->tail, 0, tail_words(e) * sizeof(long long), e->stream));
}

void split_into(vnt_engine* e, const float* x, __half* hi, __half* lo, size_t n, int op,
                int flag = vntb::kTailH16) {
  if (!e->split || !hi) return;
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(n, 256 * 4), 148 * 16);
  k_split16<<<blocks, 256, 0, e->stream>>>(x, twin_of(e, hi, lo, op, flag), n);
  VNT_LAUNCH_CHECK();
  e->launches++;
}

void node_pad(vnt_engine* e);

// Target of every split-fp16 scale: max|x| 2^sigma in [2^12, 2^13).
int h16_sigma_for(float m) { return 12 - (int)std::floor(std::log2((double)m)); }

// max |w| over the weight matrices (fp32 copies), host side.
__global__ void k_absmax(const float* __restrict__ x, size_t n, unsigned long long* out) {
  float m = 0.f;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
    m = vntb::fmax_nan(m, fabsf(x[k]));
  const unsigned b = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
  if ((threadIdx.x & 31) == 0 && b) atomicMax(out, (unsigned long long)b);
}

// Weight twins from the fp32 copies (set_params, resize, a re-split): sigma_W
// from the current max|w| first (the only operand whose max is known before
// its twins are written).
void resplit_weight_twins(vnt_engine* e);
void split_weights(vnt_engine* e) {
  if (e->node_path) node_pad(e);
  if (!e->split) return;
  const int op = h16_op_w(e);
  VNT_CUDA(cudaMemsetAsync(e->d_word, 0, sizeof(long long), e->stream));
  for (int l = 0; l < e->L; ++l) {
    if (!e->tc_layer[l]) continue;
    const size_t n = e->widths[l] * e->widths[l + 1];
    k_absmax<<<(unsigned)std::min<size_t>(ceil_div(n, 256 * 8), 1024), 256, 0, e->stream>>>(
        e->w32 + e->woff[l], n, reinterpret_cast<unsigned long long*>(e->d_word));
    VNT_LAUNCH_CHECK();
  }
  unsigned long long bits = 0;
  VNT_CUDA(cudaMemcpyAsync(&bits, e->d_word, sizeof bits, cudaMemcpyDeviceToHost, e->stream));
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  float m;
  const uint32_t b32 = (uint32_t)bits;
  std::memcpy(&m, &b32, sizeof m);
  if (!std::isfinite(m)) throw EngineError(VNT_ERR_NONFINITE, "non-finite weight");
  // the same band rule as h16_retune: sigma_W is a function of the weights'
  // history, not of when the twins were last re-split (refresh, regroup)
  const double x = std::ldexp((double)m, e->h16_sig[op]);
  if (m > 0.f && !(x >= 1024.0 && x < 16384.0)) e->h16_sig[op] = h16_sigma_for(m);
  e->h_sp->h16_mul[op] = std::ldexp(1.f, e->h16_sig[op]);
  e->h_sp->h16_inv[op] = std::ldexp(1.f, -e->h16_sig[op]);
  copy_step_params(e);
  resplit_weight_twins(e);
}

// Weight twins of the tcgen05 layers from the fp32 copies at the current sigma_W.
void resplit_weight_twins(vnt_engine* e) {
  const int op = h16_op_w(e);
  for (int l = 0; l < e->L; ++l) {
    if (!e->tc_layer[l]) continue;
    const size_t n = e->widths[l] * e->widths[l + 1];
    split_into(e, e->w32 + e->woff[l], e->w32h + e->woff[l], e->w32l + e->woff[l], n, op, vntb::kTailH16W);
  }
}

// Skinny-layer (out <= 32) kernels: NO is the compile-time bound.
template <template <int> class F, class... A>
void dispatch_skinny(int no, A&&... a) {
  if (no <= 4) F<4>::run(a...);
  else if (no <= 8) F<8>::run(a...);
  else if (no <= 12) F<12>::run(a...);
  else if (no <= 16) F<16>::run(a...);
  else F<32>::run(a...);
}

// W^T of a skinny layer fits in shared memory: the persistent resident-W kernel.
constexpr size_t kSkinnyResidentSmem = 200 * 1024;
template <int NO>
struct FwdSkinny {
  static void run(cudaStream_t s, int sms, const float* X, int K, const float* WT, int no, const float* b,
                  int rows, int act, int last, float* out) {
    const size_t smem = (size_t)no * K * sizeof(float);
    if (K % 4 == 0 && smem <= kSkinnyResidentSmem) {
      static bool attr = false;
      if (!attr) {
        VNT_CUDA(cudaFuncSetAttribute(k_fwd_skinny_res<NO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSkinnyResidentSmem));
        attr = true;
      }
      const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(sms, ceil_div(rows, 64)));
      k_fwd_skinny_res<NO><<<grid, 512, smem, s>>>(X, K, WT, no, b, rows, act, last, out);
      return;
    }
    k_fwd_skinny<NO><<<(unsigned)ceil_div(rows, 8 * skinny_rows<NO>()), 256, 0, s>>>(
        X, K, WT, no, b, rows, act, last, out);
  }
};
template <int NO>
struct BackSkinny {
  static void run(cudaStream_t s, const float* X, const float* Dn, const float* W, int in, int no, int act,
                  const int* row0, const int* nrows, int nn, float* Dout, vntb::Twin16 twins,
                  const float* scale_w, long long* Gw, int tw, const float* scale_b, long long* Gb, int tb,
                  float lim, long long* tail) {
    static const bool bulk = !(getenv("VNT_SKINNY_BULK") && getenv("VNT_SKINNY_BULK")[0] == '0');
    if (bulk && in % 4 == 0) {   // X rows streamed through smem by bulk copies (same bits)
      vntb::launch_skinny_backward_bulk<NO>(s, X, Dn, W, in, no, act, row0, nrows, nn, Dout, twins, scale_w, Gw,
                                            tw, scale_b, Gb, tb, lim, tail);
      return;
    }
    if (in % 2 == 0) {   // two features per thread (same bits)
      dim3 grid((unsigned)ceil_div(in, 256), (unsigned)nn);
      k_skinny_backward2<NO><<<grid, 128, 0, s>>>(X, Dn, W, in, no, act, row0, nrows, Dout, twins, scale_w, Gw,
                                                  tw, scale_b, Gb, tb, lim, tail);
      return;
    }
    dim3 grid((unsigned)ceil_div(in, 128), (unsigned)nn);
    k_skinny_backward<NO><<<grid, 128, 0, s>>>(X, Dn, W, in, no, act, row0, nrows, Dout, twins, scale_w, Gw,
                                               tw, scale_b, Gb, tb, lim, tail);
  }
};
template <int NO>
struct BwdSkinny {
  static void run(cudaStream_t s, const float* Dn, const float* W, int no, int in, int rows,
                  int act, const float* Xprev, float* Dout, vntb::Twin16 twins) {
    static const int chunks = [] {   // 32-row chunks per CTA (VNT_BWD_SKINNY_CHUNKS)
      const char* v = getenv("VNT_BWD_SKINNY_CHUNKS");
      return v ? std::max(1, atoi(v)) : 4;
    }();
    dim3 grid((unsigned)ceil_div(in, 32), (unsigned)ceil_div(rows, 32 * chunks)), block(32, 8);
    k_bwd_skinny<NO><<<grid, block, 0, s>>>(Dn, W, no, in, rows, act, Xprev, Dout, twins, chunks);
  }
};
template <int NO>
struct DwSkinny {
  static void run(cudaStream_t s, const float* X, int in, const float* Dn, int no, const int* row0,
                  const int* nrows, int nn, const float* scale, float lim, long long* G,
                  long long* tail, int tensor) {
    dim3 grid((unsigned)ceil_div(in, 128), (unsigned)nn);
    k_dw_skinny<NO><<<grid, 128, 0, s>>>(X, in, Dn, no, row0, nrows, scale, lim, G, tail, tensor);
  }
};

// ---------------------------------------------------------------- one pass
// Host side of observe_batch/combine for one pass: advances the device counts
// (double ops of model.cpp:123-139) and stages the per-node combine factors in
// pinned memory at `off`; the launches read them through a memcpy node.
struct StatsLaunch {
  int dev;
  size_t off;
  int n;
};

std::vector<StatsLaunch> prep_stats(vnt_engine* e, const Pass& p, size_t& off) {
  std::vector<std::vector<CombineStep>> per_dev(e->devs.size());
  for (size_t k = 0; k < p.nodes.size(); ++k) {
    auto& d = e->devs[p.nodes[k].dev];
    const double other = (double)p.nodes[k].rows;
    CombineStep st{(int)k, 0, 0.0, 0.0};
    if (d.count == 0) {
      st.copy = 1;
      d.count = other;
    } else {
      const double n = d.count + other;
      st.f1 = d.count * other / n;
      st.f2 = other / n;
      d.count = n;
    }
    per_dev[p.nodes[k].dev].push_back(st);
  }
  std::vector<StatsLaunch> out;
  for (size_t dv = 0; dv < per_dev.size(); ++dv) {
    if (per_dev[dv].empty()) continue;
    std::memcpy(e->h_combine + off, per_dev[dv].data(), per_dev[dv].size() * sizeof(CombineStep));
    out.push_back({(int)dv, off, (int)per_dev[dv].size()});
    off += per_dev[dv].size();
  }
  return out;
}

void stage_inputs_to(vnt_engine* e, const Pass& p, const double* x, const double* y,
                     bool x_on_device, double* xdst, double* ydst, cudaStream_t s) {
  const uint64_t in = e->widths[0], out = e->widths[e->L];
  const cudaMemcpyKind kind = x_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // Batch::slice copies (data.cpp:36-48): each node's contiguous rows; runs of
  // nodes adjacent both in the source batch and in the pass move as one copy.
  for (size_t k = 0; k < p.nodes.size();) {
    const auto& first = p.nodes[k];
    uint64_t nrow = first.rows;
    size_t j = k + 1;
    while (j < p.nodes.size() && p.nodes[j].src_row == first.src_row + nrow &&
           p.nodes[j].prow == first.prow + nrow) {
      nrow += p.nodes[j].rows;
      ++j;
    }
    VNT_CUDA(cudaMemcpyAsync(xdst + first.prow * in, x + first.src_row * in,
                             nrow * in * sizeof(double), kind, s));
    VNT_CUDA(cudaMemcpyAsync(ydst + first.prow * out, y + first.src_row * out,
                             nrow * out * sizeof(double), kind, s));
    k = j;
  }
}

void stage_inputs(vnt_engine* e, const Pass& p, const double* x, const double* y, bool x_on_device) {
  stage_inputs_to(e, p, x, y, x_on_device, e->xin, e->yin, e->stream);
}

std::vector<PassNode> local_nodes(vnt_engine* e, const uint64_t* node_sizes,
                                  const int32_t* node_device, uint32_t total_nodes,
                                  uint64_t batch_rows);
std::vector<Pass>& plan_for(vnt_engine* e, const std::vector<PassNode>& local);

// Copy the rows this process needs from (x, y) into the spare input buffer on
// the copy stream (single-pass plans only: multi-pass steps stage per pass).
std::vector<int64_t> staging_layout(const std::vector<PassNode>& local) {
  std::vector<int64_t> k;
  k.reserve(local.size() * 4);
  for (const auto& n : local) {
    k.push_back(n.node);
    k.push_back(n.dev);
    k.push_back((int64_t)n.rows);
    k.push_back((int64_t)n.src_row);
  }
  return k;
}

void start_prefetch(vnt_engine* e, const double* x, const double* y, uint64_t batch_rows,
                    const uint64_t* node_sizes, const int32_t* node_device, uint32_t total_nodes,
                    bool on_device, bool may_grow) {
  e->pf.valid = false;
  auto local = local_nodes(e, node_sizes, node_device, total_nodes, batch_rows);
  if (local.empty()) return;
  auto& passes = plan_for(e, local);
  if (passes.size() != 1) return;
  const Pass& p = passes[0];
  const bool fits = p.rows <= e->cap_rows && p.nodes.size() <= e->cap_vns;
  if (!fits && !may_grow) return;   // never reallocate under a running step
  ensure_capacity(e, p.rows, p.nodes.size());
  const int b = 1 - e->cur;
  stage_inputs_to(e, p, x, y, on_device, e->xbuf[b], e->ybuf[b], e->copy_stream);
  VNT_CUDA(cudaEventRecord(e->pf_event, e->copy_stream));
  e->pf.x = x;
  e->pf.y = y;
  e->pf.buf = b;
  e->pf.layout = staging_layout(local);
  e->pf.valid = true;
}

// After a step has launched its work: start the queued next batch's copy.
void start_queued_prefetch(vnt_engine* e) {
  auto& q = e->pf_next;
  if (!q.valid || e->pf.valid) return;
  q.valid = false;
  start_prefetch(e, q.x, q.y, q.rows, q.sizes.data(), q.devs.data(), (uint32_t)q.sizes.size(),
                 q.on_device, false);
}

// Use a prefetched batch if it matches (x, y) and was staged for the same
// rows (mapping, node sizes, devices): switch the staging buffer and order the
// compute stream after the copy.  Returns true if consumed.
bool take_prefetch(vnt_engine* e, const double* x, const double* y,
                   const std::vector<PassNode>& local) {
  const bool hit = e->pf.valid && e->pf.x == x && e->pf.y == y &&
                   e->pf.layout == staging_layout(local);
  e->pf.valid = false;
  if (!hit) return false;
  e->cur = e->pf.buf;
  e->xin = e->xbuf[e->cur];
  e->yin = e->ybuf[e->cur];
  VNT_CUDA(cudaStreamWaitEvent(e->stream, e->pf_event, 0));
  return true;
}

// Shared-memory floats per row of the whole-node kernel: activations of every
// layer plus deltas padded to kNodeOC (+3 for the float4 alignment of the deltas).
uint64_t node_row_floats(const vnt_engine* e) {
  uint64_t f = 4;
  for (int l = 0; l <= e->L; ++l) {
    f += e->widths[l];
    if (l > 0) f += (uint64_t)node_ld((int)e->widths[l]);
  }
  return f;
}

// Padded weight image (float4 multiple) + float4 over-read slack + alignment.
uint64_t node_wpad_floats(const vnt_engine* e) {
  int w[kNodeMaxLayers + 1] = {};
  for (int l = 0; l <= e->L && l <= kNodeMaxLayers; ++l) w[l] = (int)e->widths[l];
  return (uint64_t)node_wpad_offset(w, std::min(e->L, kNodeMaxLayers));
}
uint64_t node_wt_floats(const vnt_engine* e) { return node_wpad_floats(e) + 20; }

void node_pad(vnt_engine* e) {
  int w[kNodeMaxLayers + 1] = {};
  for (int l = 0; l <= e->L; ++l) w[l] = (int)e->widths[l];
  for (int l = 0; l < e->L; ++l) {
    const int K = w[l], N = w[l + 1];
    k_node_pad<<<(unsigned)std::min<uint64_t>(ceil_div((uint64_t)K * N, 256), 256), 256, 0,
                 e->stream>>>(e->w32 + e->woff[l], e->wpad + node_wpad_offset(w, l), K, N);
    VNT_LAUNCH_CHECK();
  }
}

// LayerStats::combine of each device's nodes into its lineage (ascending node id).
void combine_stats(vnt_engine* e, const std::vector<StatsLaunch>& stats, cudaStream_t s) {
  const uint64_t in = e->widths[0];
  for (const auto& sl : stats) {
    // the host-computed factors are read in place from pinned, mapped memory
    k_stats_combine<<<(unsigned)ceil_div(in, 128), 128, 0, s>>>(
        e->devs[sl.dev].mean, e->devs[sl.dev].m2, (int)in, e->vn_mean, e->vn_m2,
        e->m_combine + sl.off, sl.n);
    VNT_LAUNCH_CHECK();
    e->launches++;
  }
}

void backup_stats(vnt_engine* e, cudaStream_t s);
void layer_collective(vnt_engine* e, int l);
void join_stats(vnt_engine* e);
void issue_pending_gathers(vnt_engine* e);
void await_layer_weights(vnt_engine* e, int l);

// Input statistics of a pass depend on x only: observe_batch per node then the
// Chan combine into each device lineage in ascending node id
// (virtual_exec.cpp:137-138, model.cpp:152-154) run on the side stream, forked
// here; the caller joins (cudaStreamWaitEvent on join_ev) before xin changes or
// the step ends.
void fork_stats(vnt_engine* e, const Pass& p, const std::vector<StatsLaunch>& stats,
                bool side = true) {
  const size_t nn = p.nodes.size();
  const int* row0 = p.d_meta + p.rows;
  cudaStream_t st = side ? e->aux_stream : e->stream;
  if (side) {
    VNT_CUDA(cudaEventRecord(e->fork_ev, e->stream));
    VNT_CUDA(cudaStreamWaitEvent(e->aux_stream, e->fork_ev, 0));
  }
  if (!e->stats_backed) backup_stats(e, st);
  dim3 grid((unsigned)ceil_div(e->widths[0], 128), (unsigned)nn);
  k_vn_stats<<<grid, 128, 0, st>>>(e->xin, (int)e->widths[0], row0, row0 + nn, e->vn_mean,
                                   e->vn_m2);
  VNT_LAUNCH_CHECK();
  e->launches++;
  combine_stats(e, stats, st);
  VNT_CUDA(cudaEventRecord(e->join_ev, st));
}

bool stats_side_branch_layered() {
  static const bool on = getenv("VNT_STATS_BRANCH") && getenv("VNT_STATS_BRANCH")[0] == '1';
  return on;
}

// Whole-node path, single pass: step parameters, zeroed G/tail/max|g| and the
// resident batch in one launch (what copy_step_params + begin_round_device +
// launch_stage_rows do in three or more).
void step_prologue(vnt_engine* e, const Pass& p, bool stage) {
  const size_t nn = p.nodes.size();
  const int* row0 = p.d_meta + p.rows;
  uint64_t maxrows = 1;
  for (const auto& pn : p.nodes) maxrows = std::max<uint64_t>(maxrows, pn.rows);
  const unsigned slices = stage ? (unsigned)std::min<uint64_t>(
      64, ceil_div(maxrows * (e->widths[0] + e->widths[e->L]) * sizeof(double), 16384)) : 4;
  k_step_prologue<<<dim3(stage ? (unsigned)nn : 16u, slices), 256, 0, e->stream>>>(
      e->m_sp, e->d_sp, e->G, e->tail_off + tail_words(e), stage ? 1 : 0, e->xin, e->yin, row0,
      row0 + nn, row0 + 3 * nn, (int)e->widths[0], (int)e->widths[e->L]);
  VNT_LAUNCH_CHECK();
  e->launches++;
}

void launch_stage_rows(vnt_engine* e, const Pass& p) {
  const size_t nn = p.nodes.size();
  const int* row0 = p.d_meta + p.rows;
  // ~16 KB per CTA: enough CTAs in flight for the copy to run at bandwidth
  uint64_t maxrows = 1;
  for (const auto& pn : p.nodes) maxrows = std::max<uint64_t>(maxrows, pn.rows);
  const unsigned slices = (unsigned)std::min<uint64_t>(
      64, ceil_div(maxrows * (e->widths[0] + e->widths[e->L]) * sizeof(double), 16384));
  k_stage_rows<<<dim3((unsigned)nn, slices), 256, 0, e->stream>>>(e->d_sp, e->xin, e->yin, row0, row0 + nn,
                                                    row0 + 3 * nn, (int)e->widths[0],
                                                    (int)e->widths[e->L]);
  VNT_LAUNCH_CHECK();
  e->launches++;
}

// Small models: one k_node_step CTA per node does the whole pass.
void run_node_pass(vnt_engine* e, const Pass& p, const std::vector<StatsLaunch>* stats) {
  const size_t nn = p.nodes.size();
  const int* row0 = p.d_meta + p.rows;
  const int* nrows = row0 + nn;
  NodeArgs a{};
  a.x = e->xin;
  a.y = e->yin;
  a.row0 = row0;
  a.nrows = nrows;
  a.w32 = e->w32;
  a.wpad = e->wpad;
  a.wpad_floats = (int)node_wpad_floats(e);
  a.L = e->L;
  for (int l = 0; l <= e->L; ++l) a.w[l] = (int)e->widths[l];
  a.nstrips = 0;
  for (int l = 0; l < e->L; ++l) {
    a.woff[l] = (int)e->woff[l];
    a.boff[l] = (int)e->boff[l];
    a.nstrips += (int)((e->widths[l] + 1) * ceil_div(e->widths[l + 1], (uint64_t)kNodeOC));
  }
  a.act = e->act;
  a.loss = e->loss;
  uint64_t maxrows = 1;
  for (const auto& pn : p.nodes) maxrows = std::max<uint64_t>(maxrows, pn.rows);
  // CTAs per node (rows split, strips summed over DSMEM): fixed per model at creation
  const int CL = e->node_cl;
  a.rc = (int)std::min<uint64_t>(ceil_div(maxrows, (uint64_t)CL), (uint64_t)e->node_rc_max);
  a.sp = e->d_sp;
  a.lim = pow2f(e->lim_bits);
  a.G = e->G;
  a.tail = e->tail;
  a.examples = (long long)p.examples;
  const size_t base = ((size_t)a.rc * node_row_floats(e) + node_wt_floats(e) + 8 + 3) & ~(size_t)3;
  a.part_off = (int)base;
  const size_t smem = (base + (CL > 1 ? (size_t)a.nstrips * kNodeOC : 0)) * sizeof(float);
  if (smem > 227 * 1024) throw EngineError(VNT_ERR_INTERNAL, "whole-node kernel: shared memory plan exceeded");
  static size_t smem_attr[9] = {};
  if (smem > smem_attr[CL]) {
    const void* fn = CL == 8   ? (const void*)k_node_step<8>
                     : CL == 4 ? (const void*)k_node_step<4>
                     : CL == 2 ? (const void*)k_node_step<2>
                               : (const void*)k_node_step<1>;
    VNT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(smem, 48 * 1024)));
    smem_attr[CL] = std::max<size_t>(smem, 48 * 1024);
  }
  // Input statistics depend on x only: a side-stream branch beside the node kernel.
  if (stats) fork_stats(e, p, *stats);
  if (CL == 1) {
    k_node_step<1><<<(unsigned)nn, kNodeThreads, smem, e->stream>>>(a);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nn * CL));
    cfg.blockDim = dim3(kNodeThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = e->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (CL == 8) VNT_CUDA(cudaLaunchKernelEx(&cfg, k_node_step<8>, a));
    else if (CL == 4) VNT_CUDA(cudaLaunchKernelEx(&cfg, k_node_step<4>, a));
    else VNT_CUDA(cudaLaunchKernelEx(&cfg, k_node_step<2>, a));
  }
  VNT_LAUNCH_CHECK();
  e->launches++;
  e->tail_examples += p.examples;
  // Nothing in the step reads the lineage statistics: join the branch only
  // before xin is restaged or the step's control words are read (join_stats).
  if (stats) e->stats_join_pending = true;
}

// Device work of one pass (inputs already staged in xin/yin).
void run_node_pass(vnt_engine* e, const Pass& p, const std::vector<StatsLaunch>* stats);

void run_pass(vnt_engine* e, const Pass& p, const std::vector<StatsLaunch>* stats,
              bool first_write, bool layer_comm = false) {
  if (e->node_path) {
    run_node_pass(e, p, stats);
    return;
  }
  const int L = e->L;
  const uint64_t out = e->widths[L];
  const size_t nn = p.nodes.size();
  cudaStream_t s = e->stream;
  e->last_rows.clear();
  for (const auto& n : p.nodes) e->last_rows.emplace_back(n.prow, n.rows);
  const int* valid = p.d_meta;
  const int* row0 = p.d_meta + p.rows;
  const int* nrows = row0 + nn;
  const int rows = (int)p.rows;
  {
    // A split-fp16 first layer reads only the twins (allocated iff it is one).
    const bool twins = e->Xh[0] != nullptr;
    const vntb::Twin16 tw = twins ? twin_of(e, e->Xh[0], e->Xl[0], h16_op_x(e, 0)) : vntb::Twin16{};
    k_ingest<<<(unsigned)p.rows, 128, 0, s>>>(e->xin, twins ? nullptr : e->X[0], tw, valid,
                                              (int)e->widths[0], (int)e->ld0);
    VNT_LAUNCH_CHECK();
    e->launches++;
  }
  // observe_batch + combine: beside the persistent GEMMs they would hold SMs the
  // GEMM's CTAs wait for, so on the layered path they run in line by default
  // (VNT_STATS_BRANCH=1: side stream, joined at the end of the pass)
  const bool side = stats_side_branch_layered();
  if (stats) fork_stats(e, p, *stats, side);
  // Forward (model.cpp:275-287).
  for (int l = 0; l < L; ++l) {
    const int K = (int)e->widths[l], N = (int)e->widths[l + 1];
    const bool last = (l == L - 1);
    await_layer_weights(e, l);   // sharded update: this layer's gathered weights
    const float* W = e->w32 + e->woff[l];
    const float* b = e->w32 + e->boff[l];
    prof_begin(e);
    if (e->tc_layer[l]) {
      tc_forward(e, l, rows, last);
    } else if (N <= 32) {
      dispatch_skinny<FwdSkinny>(N, s, e->sm_count, e->X[l], K, e->wt32 + e->wtoff[l], N, b, rows, e->act,
                                 last ? 1 : 0, last ? e->logits : e->X[l + 1]);
      VNT_LAUNCH_CHECK();
      e->launches++;
    } else {
      dim3 grid((unsigned)ceil_div(N, 64), (unsigned)ceil_div(p.rows, 64));
      if (last) {
        k_gemm_ffma<kEpiLogits><<<grid, 256, 0, s>>>(e->X[l], K, W, N, rows, N, K, b, e->act,
                                                     e->logits, N, nullptr, 0);
      } else {
        k_gemm_ffma<kEpiHidden><<<grid, 256, 0, s>>>(e->X[l], K, W, N, rows, N, K, b, e->act,
                                                     e->X[l + 1], N, nullptr, 0);
      }
      VNT_LAUNCH_CHECK();
      e->launches++;
    }
    prof_end(e, 2.0 * rows * (double)K * N);
    if (!last && !e->tc_layer[l])   // tcgen05 epilogues write the twins themselves
      split_into(e, e->X[l + 1], e->Xh[l + 1], e->Xl[l + 1], p.rows * (uint64_t)N, h16_op_x(e, l + 1));
  }
  VNT_CUDA(cudaEventRecord(e->ev[1], s));
  // Loss + output delta (model.cpp:289-315); pad rows get zero deltas.
  {
    const unsigned warps_per_block = 8;
    k_loss<<<(unsigned)ceil_div(p.rows, warps_per_block), warps_per_block * 32, 0, s>>>(
        e->logits, e->yin, rows, (int)out, e->loss, e->D[L], valid, e->tail, e->d_sp);
    VNT_LAUNCH_CHECK();
    e->launches++;
    split_into(e, e->D[L], e->Dh[L], e->Dl[L], p.rows * out, h16_op_d(e, L));
  }
  // Backward (model.cpp:317-338): dW/db per node into the exact sum, then delta.
  const float lim = pow2f(e->lim_bits);
  int db_done = -1;   // a fused skinny backward already produced this layer's db
  for (int l = L - 1; l >= 0; --l) {
    const int in_l = (int)e->widths[l], out_l = (int)e->widths[l + 1];
    const int tw = 2 * l, tb = 2 * l + 1;
    const bool skinny = !e->tc_layer[l] && out_l <= 32;
    prof_begin(e);
    if (e->tc_layer[l]) {
      tc_weight_grad(e, l, p, row0, nrows, sp_scale(e, tw), lim, first_write, tw);
    } else if (skinny) {
      // dW_l, D[l] (twins, plain only when a non-tcgen05 consumer needs it) and
      // the db of layer l-1 in one pass over X[l] (k_skinny_backward)
      const bool data = l > 0;
      dispatch_skinny<BackSkinny>(out_l, s, e->X[l], e->D[l + 1], e->w32 + e->woff[l], in_l, out_l, e->act,
                                  row0, nrows, (int)nn, data && !e->Dh[l] ? e->D[l] : nullptr,
                                  data && e->Dh[l] ? twin_of(e, e->Dh[l], e->Dl[l], h16_op_d(e, l))
                                                   : vntb::Twin16{},
                                  sp_scale(e, tw),
                                  e->G + e->woff[l], tw, data ? sp_scale(e, tb - 2) : nullptr,
                                  data ? e->G + e->boff[l - 1] : nullptr, tb - 2, lim, e->tail);
      VNT_LAUNCH_CHECK();
      e->launches++;
      if (data) db_done = l - 1;
    } else {
      dim3 grid((unsigned)ceil_div(out_l, 64), (unsigned)ceil_div(in_l, 64), (unsigned)nn);
      k_dw_ffma<<<grid, 256, 0, s>>>(e->X[l], e->D[l + 1], in_l, out_l, row0, nrows, sp_scale(e, tw), lim,
                                     e->G + e->woff[l], e->tail, tw);
      VNT_LAUNCH_CHECK();
      e->launches++;
    }
    prof_end(e, 2.0 * rows * (double)in_l * out_l);
    if (db_done != l) {
      // a tcgen05 bwd-data leaves D only as its split-fp16 twins
      const bool twins_only = l + 1 < L && e->tc_layer[l + 1] && e->Dh[l + 1];
      if (twins_only && out_l % 2 == 0) {
        dim3 grid((unsigned)ceil_div(out_l, 256), (unsigned)nn);
        k_db2<<<grid, 128, 0, s>>>(e->Dh[l + 1], e->Dl[l + 1], h16_inv(e, h16_op_d(e, l + 1)), out_l, row0,
                                   nrows, sp_scale(e, tb), lim, e->G + e->boff[l], e->tail, tb);
      } else {
        dim3 grid((unsigned)ceil_div(out_l, 128), (unsigned)nn);
        k_db<<<grid, 128, 0, s>>>(e->D[l + 1], twins_only ? e->Dh[l + 1] : nullptr,
                                  twins_only ? e->Dl[l + 1] : nullptr,
                                  twins_only ? h16_inv(e, h16_op_d(e, l + 1)) : nullptr,
                                  out_l, row0, nrows, sp_scale(e, tb), lim, e->G + e->boff[l], e->tail, tb);
      }
      VNT_LAUNCH_CHECK();
      e->launches++;
    }
    if (layer_comm) layer_collective(e, l);   // layer l's gradient is final in this process
    if (l > 0 && !skinny) {
      prof_begin(e);
      if (e->tc_layer[l]) {
        tc_backward_data(e, l, rows);
      } else {
        const float* WT = e->wt32 + e->wtoff[l];
        dim3 grid((unsigned)ceil_div(in_l, 64), (unsigned)ceil_div(p.rows, 64));
        k_gemm_ffma<kEpiBwd><<<grid, 256, 0, s>>>(e->D[l + 1], out_l, WT, in_l, rows, in_l, out_l,
                                                  nullptr, e->act, e->D[l], in_l, e->X[l], in_l);
        VNT_LAUNCH_CHECK();
        e->launches++;
      }
      prof_end(e, 2.0 * rows * (double)in_l * out_l);
      if (!e->tc_layer[l])   // tcgen05 epilogues write the twins themselves
        split_into(e, e->D[l], e->Dh[l], e->Dl[l], p.rows * (uint64_t)in_l, h16_op_d(e, l));
    }
  }
  if (stats) VNT_CUDA(cudaStreamWaitEvent(e->stream, e->join_ev, 0));
}

void begin_round_host(vnt_engine* e, uint64_t batch_hint) {
  e->stats_backed = false;
  e->acc_examples = 0;
  e->acc_partials = 0;
  e->tail_examples = 0;
  e->acc_started = false;
  e->round_open = true;
  if (!e->scales_init) {
    std::fill(e->scales.begin(), e->scales.end(), initial_scale(batch_hint));
    e->scales_init = true;
  }
  for (auto& d : e->devs) d.count_bak = d.count;
}

void begin_round_device(vnt_engine* e) {
  tail_reset(e);
  // Slices filled by exact int64 atomics start from zero (bias always, weights
  // of non-tcgen05 layers); tcgen05 dW tiles store on the first pass.
  if (e->node_path) {
    VNT_CUDA(cudaMemsetAsync(e->G, 0, e->P * sizeof(long long), e->stream));
  } else {
  for (int l = 0; l < e->L; ++l) {
    VNT_CUDA(cudaMemsetAsync(e->G + e->boff[l], 0, e->widths[l + 1] * sizeof(long long), e->stream));
    if (!e->tc_layer[l])
      VNT_CUDA(cudaMemsetAsync(e->G + e->woff[l], 0, e->widths[l] * e->widths[l + 1] * sizeof(long long),
                               e->stream));
  }
  }
  // lineage backups run on the statistics branch (fork_stats), before the combine
}

// Lineage statistics as of the round start (restored if the step is redone).
void backup_stats(vnt_engine* e, cudaStream_t s) {
  const uint64_t in = e->widths[0];
  for (auto& d : e->devs) {
    k_copy_f64x2<<<(unsigned)std::min<uint64_t>(ceil_div(in, 256), 64), 256, 0, s>>>(
        d.mean, d.mean_bak, d.m2, d.m2_bak, (int)in);
    VNT_LAUNCH_CHECK();
  }
  e->stats_backed = true;
}

// Collective log (vnt_engine_comm_log): every rank of a group must issue the
// identical sequence, so tests compare these across rank layouts.
enum : uint64_t {
  kLogAllReduce = 1, kLogReduceScatter = 2, kLogAllGather = 3, kLogMax = 4, kLogCount = 5,
  kLogBroadcast = 6, kLogSend = 7, kLogRecv = 8
};
void log_comm(vnt_engine* e, uint64_t op, uint64_t off, uint64_t n) {
  e->comm_log.insert(e->comm_log.end(), {op, off, n});
  if (e->comm_log.size() > 6144) e->comm_log.erase(e->comm_log.begin(), e->comm_log.begin() + 3072);
}

// Sum of a host count over the process group (blocking; first round only).
uint64_t global_count(vnt_engine* e, uint64_t local) {
  long long v = (long long)local;
  VNT_CUDA(cudaMemcpyAsync(e->d_word, &v, sizeof v, cudaMemcpyHostToDevice, e->stream));
  e->comm->allreduce_sum_i64(e->d_word, 1, e->stream);
  log_comm(e, kLogCount, 0, 1);
  VNT_CUDA(cudaMemcpyAsync(&v, e->d_word, sizeof v, cudaMemcpyDeviceToHost, e->stream));
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  return (uint64_t)v;
}

void begin_round(vnt_engine* e, uint64_t batch_hint) {
  if (e->round_open) return;
  begin_round_host(e, batch_hint);
  upload_step_params(e, 0.0, 0.0);
  begin_round_device(e);
}

// Undo the round's input-statistics updates (a rescaled redo observes again).
void restore_stats(vnt_engine* e) {
  const uint64_t in = e->widths[0];
  for (auto& d : e->devs) {
    d.count = d.count_bak;
    if (!e->stats_backed) continue;   // nothing observed this round: the lineage is untouched
    VNT_CUDA(cudaMemcpyAsync(d.mean, d.mean_bak, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
    VNT_CUDA(cudaMemcpyAsync(d.m2, d.m2_bak, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
  }
}

void accumulate(vnt_engine* e, std::vector<PassNode>& local, const double* x, const double* y,
                bool on_device, bool do_stats, bool layer_comm = false) {
  issue_pending_gathers(e);   // weights of the last sharded update, awaited per layer
  auto& passes = plan_for(e, local);
  std::vector<std::vector<StatsLaunch>> stats(passes.size());
  if (do_stats) {
    size_t total = 0;
    for (const auto& p : passes) total += p.nodes.size();
    ensure_combine(e, total);
    size_t off = 0;
    for (size_t i = 0; i < passes.size(); ++i) stats[i] = prep_stats(e, passes[i], off);
  }
  for (size_t i = 0; i < passes.size(); ++i) {
    const auto& p = passes[i];
    ensure_capacity(e, p.rows, p.nodes.size());
    join_stats(e);   // the previous pass's statistics still read xin
    // A prefetched batch is consumed on the first attempt only (on a rescale
    // retry the prefetch slot already holds the next batch).
    bool took = false;
    if (i == 0 && do_stats) {
      if (passes.size() == 1) took = take_prefetch(e, x, y, local);
      else e->pf.valid = false;
    }
    if (!took) stage_inputs(e, p, x, y, on_device);
    run_pass(e, p, do_stats ? &stats[i] : nullptr, !e->acc_started,
             layer_comm && i + 1 == passes.size());
    e->acc_started = true;
    e->acc_examples += p.examples;
    e->acc_partials += p.nodes.size();
  }
}

constexpr int kCommSms = 16;   // SMs left to NCCL while GEMMs run beside its kernels

bool overlap_wanted() {
  return !(getenv("VNT_COMM_OVERLAP") && getenv("VNT_COMM_OVERLAP")[0] == '0');
}

bool shard_wanted() { return !(getenv("VNT_SHARD") && getenv("VNT_SHARD")[0] == '0'); }

void free_shards(vnt_engine* e) {
  for (void* p : {(void*)e->Gs, (void*)e->ag_send, (void*)e->ag_recv})
    if (p) cudaFree(p);
  e->Gs = nullptr;
  e->ag_send = nullptr;
  e->ag_recv = nullptr;
  e->shard = false;
  e->ag_pending = false;
  e->ag_wait.assign(e->L, 0);
}

// This rank's fp32 chunk of every layer slice, from the current fp64 master
// (what the next all-gather sends when no update has happened since).
void refill_ag_send(vnt_engine* e) {
  for (int l = 0; l < e->L; ++l) {
    const long long n = (long long)(e->sh_hi[l] - e->sh_lo[l]);
    if (n <= 0) continue;
    k_f64_to_f32<<<(unsigned)std::min<long long>(ceil_div((uint64_t)n, 256), 1024), 256, 0, e->stream>>>(
        e->w64 + e->woff[l] + e->sh_lo[l], e->ag_send + e->sh_soff[l], n);
    VNT_LAUNCH_CHECK();
  }
}

// Shard layout of the current group: layer slice n_l = in*out + out, chunk
// c_l = ceil(n_l / G) rounded up to 32 words, rank r owns [r c_l, (r+1) c_l).
void setup_shards(vnt_engine* e) {
  free_shards(e);
  if (!e->comm || e->node_path || !shard_wanted()) return;
  const uint64_t S = (uint64_t)e->comm->size(), r = (uint64_t)e->comm->rank();
  if (S > (uint64_t)kMaxRanks) throw EngineError(VNT_ERR_CONFIG, "sharded update supports up to 64 ranks");
  e->sh_c.assign(e->L, 0);
  e->sh_lo.assign(e->L, 0);
  e->sh_hi.assign(e->L, 0);
  e->sh_soff.assign(e->L, 0);
  e->sh_aoff.assign(e->L, 0);
  uint64_t soff = 0, aoff = 0;
  for (int l = 0; l < e->L; ++l) {
    const uint64_t n = e->widths[l] * e->widths[l + 1] + e->widths[l + 1];
    const uint64_t c = round_up(ceil_div(n, S), 32);
    e->sh_c[l] = c;
    e->sh_lo[l] = std::min(r * c, n);
    e->sh_hi[l] = std::min((r + 1) * c, n);
    e->sh_soff[l] = soff;
    e->sh_aoff[l] = aoff;
    soff += c;
    aoff += S * c;
  }
  e->Gs = (long long*)dalloc(soff * sizeof(long long));
  e->ag_send = (float*)dalloc(soff * sizeof(float));
  VNT_CUDA(cudaMemset(e->ag_send, 0, soff * sizeof(float)));
  e->ag_recv = (float*)dalloc(aoff * sizeof(float));
  if (e->ag_ev.empty()) {
    e->ag_ev.assign(e->L, nullptr);
    for (auto& ev : e->ag_ev) VNT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    VNT_CUDA(cudaEventCreateWithFlags(&e->ag_fork, cudaEventDisableTiming));
  }
  e->shard = true;
  refill_ag_send(e);
}

// With a stream-ordered group (NCCL), overlap the per-layer reductions with
// the backward (and the deferred weight gathers with the forward) on a comm
// stream; GEMMs then leave kCommSms SMs to the NCCL kernels beside them.
// Host-callback groups run every collective in line.
void setup_comm(vnt_engine* e) {
  drop_graphs(e);
  e->gemm_sms = e->sm_count;
  e->comm_overlap = e->comm && e->comm->on_stream() && overlap_wanted();
  if (e->comm_overlap) {
    if (!e->comm_stream) {   // idempotent (regroup calls it again)
      VNT_CUDA(cudaStreamCreateWithFlags(&e->comm_stream, cudaStreamNonBlocking));
      e->layer_ev.assign(e->L, nullptr);
      for (auto& ev : e->layer_ev) VNT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      VNT_CUDA(cudaEventCreateWithFlags(&e->comm_ev, cudaEventDisableTiming));
    }
    e->gemm_sms = std::max(2, (e->sm_count - kCommSms) & ~1);   // even: CTA pairs
  }
  setup_shards(e);
}

void allreduce(vnt_engine* e, long long* p, size_t n, cudaStream_t s) {
  log_comm(e, kLogAllReduce, (uint64_t)(p - e->G), (uint64_t)n);
  e->comm->allreduce_sum_i64(p, n, s);
}

// Layer l's slice of G -> this rank's reduced chunk in Gs.  The send range
// G * c_l may run past the slice (into the next layer's final sums or the
// zero gap before the tail); those words land beyond n_l and are ignored.
void reduce_scatter_layer(vnt_engine* e, int l, cudaStream_t s) {
  log_comm(e, kLogReduceScatter, e->woff[l], e->sh_c[l]);
  e->comm->reduce_scatter_sum_i64(e->G + e->woff[l], e->Gs + e->sh_soff[l], e->sh_c[l], s);
}

// The step's gradient reduction, in line on the compute stream: per layer
// (reduce-scatter, sharded update) then the tail, or one all-reduce of G.
// `full`: the whole mean gradient is wanted on every rank (sync_gradients).
void collective(vnt_engine* e, bool full = false) {
  if (!e->comm) return;
  if (e->shard && !full) {
    for (int l = e->L - 1; l >= 0; --l) reduce_scatter_layer(e, l, e->stream);
    allreduce(e, e->tail, e->ntail, e->stream);
    return;
  }
  // Exact int64 sum over processes; associative, so any algorithm or topology
  // gives the same bits.
  allreduce(e, e->G, e->tail_off + e->ntail, e->stream);
}

// The split-fp16 operand maxima of this step over the group (the next step's
// scales, h16_retune, must be the same on every rank).
bool h16_reduced(const vnt_engine* e) {
  if (!e->split || e->node_path) return false;
  for (int l = 0; l < e->L; ++l)
    if (e->tc_layer[l]) return true;
  return false;
}
void h16_reduce(vnt_engine* e) {
  if (!e->comm || !h16_reduced(e)) return;
  log_comm(e, kLogMax, (uint64_t)(reinterpret_cast<long long*>(e->h16max) - e->G), h16_nops(e));
  e->comm->allreduce_max_u64(e->h16max, h16_nops(e), e->stream);
}

// Overlapped variant, issued identically (same calls, same order) on every
// rank: layer l's G slice once its dW/db are final, from the compute stream's
// point of view (run_pass records layer_ev[l] after them).
void layer_collective(vnt_engine* e, int l) {
  VNT_CUDA(cudaEventRecord(e->layer_ev[l], e->stream));
  VNT_CUDA(cudaStreamWaitEvent(e->comm_stream, e->layer_ev[l], 0));
  if (e->shard) {
    reduce_scatter_layer(e, l, e->comm_stream);
    return;
  }
  const uint64_t n = e->widths[l] * e->widths[l + 1] + e->widths[l + 1];   // W then b, contiguous
  allreduce(e, e->G + e->woff[l], n, e->comm_stream);
}

// The tail (loss, examples, flags) last, then the compute stream waits for all.
void finish_layer_collectives(vnt_engine* e) {
  VNT_CUDA(cudaEventRecord(e->layer_ev[0], e->stream));
  VNT_CUDA(cudaStreamWaitEvent(e->comm_stream, e->layer_ev[0], 0));
  allreduce(e, e->tail, e->ntail, e->comm_stream);
  VNT_CUDA(cudaEventRecord(e->comm_ev, e->comm_stream));
  VNT_CUDA(cudaStreamWaitEvent(e->stream, e->comm_ev, 0));
}

// Start the all-gathers of the weights the last sharded update produced
// (layer 0 first, so the forward can begin while the rest arrive).
void issue_pending_gathers(vnt_engine* e) {
  if (!e->shard || !e->ag_pending) return;
  cudaStream_t cs = e->comm_overlap ? e->comm_stream : e->stream;
  if (e->comm_overlap) {   // ag_send was written on the compute stream
    VNT_CUDA(cudaEventRecord(e->ag_fork, e->stream));
    VNT_CUDA(cudaStreamWaitEvent(e->comm_stream, e->ag_fork, 0));
  }
  for (int l = 0; l < e->L; ++l) {
    log_comm(e, kLogAllGather, e->woff[l], e->sh_c[l]);
    e->comm->allgather(e->ag_send + e->sh_soff[l], e->ag_recv + e->sh_aoff[l], e->sh_c[l] * sizeof(float), cs);
    if (e->comm_overlap) VNT_CUDA(cudaEventRecord(e->ag_ev[l], cs));
  }
  e->ag_wait.assign(e->L, 1);
  e->ag_pending = false;
}

// Before layer l's fp32 weights are read: wait for its gather and expand it
// into the copies the kernels read (same outputs as launch_sgd's unsharded path).
void await_layer_weights(vnt_engine* e, int l) {
  if (!e->shard || !e->ag_wait[l]) return;
  cudaStream_t s = e->stream;
  if (e->comm_overlap) VNT_CUDA(cudaStreamWaitEvent(s, e->ag_ev[l], 0));
  const float* src = e->ag_recv + e->sh_aoff[l];
  const int rows = (int)e->widths[l], cols = (int)e->widths[l + 1];
  const bool twins_only = e->split && e->tc_layer[l];
  const uint64_t wo = e->woff[l], to = e->wtoff[l], bo = e->boff[l];
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32)), block(32, 8);
  // the twins feed this step: their range flag is the redo slot kTailH16
  const vntb::Twin16 tw = twins_only ? twin_of(e, e->w32h + wo, e->w32l + wo, h16_op_w(e)) : vntb::Twin16{};
  k_expand_weight<<<grid, block, 0, s>>>(src, rows, cols, twins_only ? nullptr : e->w32 + wo,
                                         e->tc_layer[l] ? nullptr : e->wt32 + to, tw);
  VNT_LAUNCH_CHECK();
  k_expand_vec<<<(unsigned)ceil_div(cols, 256), 256, 0, s>>>(src + (size_t)rows * cols, cols, e->w32 + bo);
  VNT_LAUNCH_CHECK();
  e->launches += 2;
  e->ag_wait[l] = 0;
}

// Every fp32 weight current (before an unsharded update, a regroup, ...).
void flush_gathers(vnt_engine* e) {
  issue_pending_gathers(e);
  for (int l = 0; l < e->L; ++l) await_layer_weights(e, l);
}

// Every rank's fp64 master (and momentum) complete: all-gather the shards
// (get_params, regroup, unsharded updates).  Blocking; not on the hot path.
void gather_master(vnt_engine* e) {
  if (!e->shard || e->master_valid) return;
  const uint64_t S = (uint64_t)e->comm->size();
  uint64_t cmax = 0;
  for (int l = 0; l < e->L; ++l) cmax = std::max(cmax, e->sh_c[l]);
  double* send = (double*)dalloc(cmax * sizeof(double));
  double* recv = (double*)dalloc(S * cmax * sizeof(double));
  for (double* m : {e->w64, e->v64}) {
    if (!m) continue;
    for (int l = 0; l < e->L; ++l) {
      const uint64_t n = e->widths[l] * e->widths[l + 1] + e->widths[l + 1];
      const uint64_t c = e->sh_c[l], own = e->sh_hi[l] - e->sh_lo[l];
      VNT_CUDA(cudaMemsetAsync(send, 0, c * sizeof(double), e->stream));
      if (own)
        VNT_CUDA(cudaMemcpyAsync(send, m + e->woff[l] + e->sh_lo[l], own * sizeof(double),
                                 cudaMemcpyDeviceToDevice, e->stream));
      log_comm(e, kLogAllGather, e->woff[l], c);
      e->comm->allgather(send, recv, c * sizeof(double), e->stream);
      VNT_CUDA(cudaMemcpyAsync(m + e->woff[l], recv, n * sizeof(double), cudaMemcpyDeviceToDevice,
                               e->stream));
    }
  }
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  cudaFree(send);
  cudaFree(recv);
  e->master_valid = true;
}

// Sharded update: this rank's chunk of every layer, then the per-tensor
// max|g| (the next step's scales) is max-reduced over the group.
void launch_sgd_shard(vnt_engine* e, bool reduce_h16) {
  cudaStream_t s = e->stream;
  if (reduce_h16) h16_reduce(e);   // the update's range check reads the group's maxima
  for (int l = 0; l < e->L; ++l) {
    ShardSgdArgs a{};
    a.h16max = e->h16max;
    a.h16n = h16_reduced(e) ? h16_nops(e) : 0;
    a.Gs = e->Gs + e->sh_soff[l];
    a.w64 = e->w64 + e->woff[l];
    a.v64 = e->v64 ? e->v64 + e->woff[l] : nullptr;
    a.out32 = e->ag_send + e->sh_soff[l];
    a.gmax = e->gmax + 2 * l;
    a.tail = e->tail;
    a.ntail_flags = (int)ntensors(e);
    a.sp = e->d_sp;
    a.tw = 2 * l;
    a.lo = (long long)e->sh_lo[l];
    a.hi = (long long)e->sh_hi[l];
    a.nw = (long long)(e->widths[l] * e->widths[l + 1]);
    const uint64_t n = std::max<uint64_t>(1, e->sh_hi[l] - e->sh_lo[l]);
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(n, 256 * 4), (uint64_t)e->sm_count * 8);
    if (a.v64) k_sgd_shard<true><<<grid, 256, 0, s>>>(a);
    else k_sgd_shard<false><<<grid, 256, 0, s>>>(a);
    VNT_LAUNCH_CHECK();
    e->launches++;
  }
  log_comm(e, kLogMax, (uint64_t)(reinterpret_cast<long long*>(e->gmax) - e->G), ntensors(e));
  e->comm->allreduce_max_u64(e->gmax, ntensors(e), s);
  e->ag_pending = true;
  e->master_valid = false;
}

// Copy this rank's chunks out of an all-reduced G (the unsharded
// sync_gradients path) so a sharded update can follow.
void load_shards_from_full(vnt_engine* e) {
  for (int l = 0; l < e->L; ++l) {
    const uint64_t own = e->sh_hi[l] - e->sh_lo[l];
    if (own)
      VNT_CUDA(cudaMemcpyAsync(e->Gs + e->sh_soff[l], e->G + e->woff[l] + e->sh_lo[l],
                               own * sizeof(long long), cudaMemcpyDeviceToDevice, e->stream));
  }
}

// lr, 1/B (virtual_exec.cpp:165), momentum and 2^-s come from the step params.
// reduce_h16: max-reduce the split-fp16 operand maxima first (every path
// except an sgd_apply after vnt_engine_sync, which already did).
void launch_sgd(vnt_engine* e, bool reduce_h16 = true) {
  if (e->shard) {
    launch_sgd_shard(e, reduce_h16);
    return;
  }
  if (reduce_h16) h16_reduce(e);
  cudaStream_t s = e->stream;
  if (e->node_path) {   // all tensors in one launch, row-major fp32 copies only
    SgdMulti m{};
    uint64_t maxn = 1;
    for (int t = 0; t < (int)ntensors(e); ++t) {
      const int l = t / 2;
      SgdArgs& a = m.t[t];
      const uint64_t off = (t & 1) ? e->boff[l] : e->woff[l];
      a.w64 = e->w64 + off;
      a.v64 = e->v64 ? e->v64 + off : nullptr;
      a.G = e->G + off;
      a.w32 = e->w32 + off;
      a.gout = e->gout ? e->gout + off : nullptr;
      a.gmax = e->gmax + t;
      a.tail = e->tail;
      a.ntail_flags = (int)ntensors(e);
      a.sp = e->d_sp;
      a.tensor = t;
      a.rows = (t & 1) ? 1 : (int)e->widths[l];
      a.cols = (int)e->widths[l + 1];
      if (!(t & 1)) {
        int w[kNodeMaxLayers + 1] = {};
        for (int k = 0; k <= e->L; ++k) w[k] = (int)e->widths[k];
        a.wpad = e->wpad + node_wpad_offset(w, l);
        a.ldw = node_ldw(a.cols);
      }
      maxn = std::max<uint64_t>(maxn, (uint64_t)a.rows * a.cols);
    }
    dim3 grid((unsigned)std::min<uint64_t>(ceil_div(maxn, 256), 64), (unsigned)ntensors(e));
    k_sgd_multi<<<grid, 256, 0, s>>>(m);
    VNT_LAUNCH_CHECK();
    e->launches++;
    return;
  }
  // bias vectors: k_sgd_multi, one grid row per tensor (the same per-element
  // update, sgd_one), instead of a launch per layer
  SgdMulti biases{};
  int nb = 0;
  uint64_t maxb = 1;
  auto flush_biases = [&] {
    if (!nb) return;
    dim3 grid((unsigned)std::min<uint64_t>(ceil_div(maxb, 256), 64), (unsigned)nb);
    k_sgd_multi<<<grid, 256, 0, s>>>(biases);
    VNT_LAUNCH_CHECK();
    e->launches++;
    nb = 0;
    maxb = 1;
  };
  for (int l = 0; l < e->L; ++l) {
    for (int part = 0; part < 2; ++part) {
      const int t = 2 * l + part;
      SgdArgs a{};
      const uint64_t off = part ? e->boff[l] : e->woff[l];
      a.w64 = e->w64 + off;
      a.v64 = e->v64 ? e->v64 + off : nullptr;
      a.G = e->G + off;
      // a split-fp16 layer's weight GEMMs read only the twins (written for
      // the next step: their range flag is kTailH16W, not a redo of this one)
      // Wᵀ (fp32) only for a non-tcgen05 layer (the skinny / FFMA forward)
      const bool twins_only = part == 0 && e->split && e->tc_layer[l];
      a.w32 = twins_only ? nullptr : e->w32 + off;
      a.wt32 = (part || e->tc_layer[l]) ? nullptr : e->wt32 + e->wtoff[l];
      if (twins_only) {
        a.w32h = e->w32h + off;
        a.w32l = e->w32l + off;
        a.wtw = twin_of(e, a.w32h, a.w32l, h16_op_w(e), vntb::kTailH16W);
      }
      a.gout = e->gout ? e->gout + off : nullptr;
      a.gmax = e->gmax + t;
      a.tail = e->tail;
      a.ntail_flags = (int)ntensors(e);
      a.sp = e->d_sp;
      a.h16max = e->h16max;
      a.h16n = h16_reduced(e) ? h16_nops(e) : 0;
      a.tensor = t;
      if (part == 0) {
        a.rows = (int)e->widths[l];
        a.cols = (int)e->widths[l + 1];
        // rows per tile: 32 measured best on cfg3 (4.7 TB/s vs 4.4 at 64, 3.3 at 128)
        static const int tr = getenv("VNT_SGD_TR") ? atoi(getenv("VNT_SGD_TR")) : 32;
        const int TR = (tr == 64 || tr == 128) ? tr : 32;
        dim3 grid((unsigned)ceil_div(a.cols, 32), (unsigned)ceil_div(a.rows, TR)), block(32, 8);
        if (twins_only && a.rows % 2 == 0 && a.cols % 2 == 0) {
          dim3 g2((unsigned)ceil_div(a.cols, 64), (unsigned)ceil_div(a.rows, 64));
          if (a.v64) k_sgd_twins<true><<<g2, block, 0, s>>>(a);
          else k_sgd_twins<false><<<g2, block, 0, s>>>(a);
        } else if (a.v64) k_sgd_weight<true><<<grid, block, 0, s>>>(a);
        else if (TR == 32) k_sgd_weight<false, 32><<<grid, block, 0, s>>>(a);
        else if (TR == 128) k_sgd_weight<false, 128><<<grid, block, 0, s>>>(a);
        else k_sgd_weight<false><<<grid, block, 0, s>>>(a);
      } else {
        // the biases of up to 2 kNodeMaxLayers layers in one launch (below)
        a.rows = 1;
        a.cols = (int)e->widths[l + 1];
        biases.t[nb++] = a;
        maxb = std::max<uint64_t>(maxb, (uint64_t)a.cols);
        if (nb == 2 * kNodeMaxLayers || l == e->L - 1) flush_biases();
        continue;
      }
      VNT_LAUNCH_CHECK();
      e->launches++;
    }
  }
  flush_biases();
}

struct Readback {
  double loss_sum;
  uint64_t examples;
  uint64_t partials;
  bool nonfinite;
  bool loss_range;             // a row loss outside the int64 range at this quantum
  bool h16_range;              // a split-fp16 operand of this step left its range (redo)
  std::vector<int> overflow;   // tensor ids
};

// The statistics side branch of a whole-node pass, joined lazily.
void join_stats(vnt_engine* e) {
  if (!e->stats_join_pending) return;
  VNT_CUDA(cudaStreamWaitEvent(e->stream, e->join_ev, 0));
  e->stats_join_pending = false;
}

void enqueue_readback(vnt_engine* e, bool with_gmax) {
  join_stats(e);   // the step ends here: its statistics branch must have finished
  cudaStream_t s = e->stream;
  k_copy_words<<<1, 64, 0, s>>>(reinterpret_cast<const unsigned long long*>(e->tail),
                                reinterpret_cast<unsigned long long*>(e->m_tail),
                                (int)(with_gmax || e->split ? tail_words(e) : e->ntail));
  VNT_LAUNCH_CHECK();
}

Readback parse_readback(vnt_engine* e) {
  Readback r;
  r.loss_sum = std::ldexp((double)e->h_tail[kTailLoss], -e->loss_bits);
  r.examples = (uint64_t)e->h_tail[kTailExamples];
  r.partials = (uint64_t)e->h_tail[kTailPartials];
  r.nonfinite = e->h_tail[kTailNonfinite] != 0;
  r.loss_range = e->h_tail[kTailLossRange] != 0;
  r.h16_range = e->split && e->h_tail[kTailH16] != 0;
  for (uint32_t t = 0; t < ntensors(e); ++t)
    if (e->h_tail[kTailOverflow + t]) r.overflow.push_back((int)t);
  return r;
}

Readback read_tail(vnt_engine* e, bool with_gmax) {
  enqueue_readback(e, with_gmax);
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  return parse_readback(e);
}

// Back to the default loss quantum once the mean row loss is 2^8 below the
// range of the default (a function of global values: identical on every rank).
void relax_loss_bits(vnt_engine* e, double mean_loss) {
  if (e->loss_bits >= kLossScaleBits) return;
  if (std::fabs(mean_loss) * std::ldexp(1.0, kLossScaleBits + 8) < std::ldexp(1.0, 62) / e->loss_rows)
    e->loss_bits = kLossScaleBits;
}

void refresh_from_master(vnt_engine* e);

// Split-fp16 scales for the next step (or the redo) from this step's max|x|
// per operand — max-reduced over the group, so identical on every rank.  An
// operand whose max|x| 2^sigma left [2^10, 2^14) is re-targeted to [2^12,
// 2^13) (h16_sigma_for).  The weight twins the update just wrote (unsharded)
// are re-split from the fp64 master at the new sigma; sharded, the next
// weight expansion reads it.  Returns false if some operand max is not finite.
struct H16Review {
  bool finite = true;   // every operand max finite
  bool under = false;   // some max|x| 2^sigma < kH16Under: the device skipped the update
};
H16Review h16_retune(vnt_engine* e) {
  H16Review r;
  if (!e->split) return r;
  auto max_of = [&](int op) {
    const uint32_t b = (uint32_t)e->h_h16max[op];
    float m;
    std::memcpy(&m, &b, sizeof m);
    return m;
  };
  // one operand's band rule; returns false past an fp16 overflow
  auto retune = [&](int op) {
    const float m = max_of(op);
    const double x = std::ldexp((double)m, e->h16_sig[op]);
    // the device-side test of block_poisoned (StepParams mul < 2^100)
    if (h16_reduced(e) && x < vntb::kH16Under && e->h16_sig[op] < vntb::kH16SigMax) r.under = true;
    if (!(x >= 1024.0 && x < 16384.0)) e->h16_sig[op] = std::min(h16_sigma_for(m), vntb::kH16SigMax);
    return x < (double)vntb::kH16Lim;
  };
  // Activations and deltas in dataflow order (X0 .. X_L, then D_L .. D_1): an
  // operand that overflowed fp16 poisons everything computed from it, so the
  // scan stops there (the redo measures the rest); a non-finite maximum before
  // any overflow is a genuine non-finite value.
  std::vector<int> order;
  for (int l = 0; l <= e->L; ++l) order.push_back(h16_op_x(e, l));
  for (int l = e->L; l >= 1; --l) order.push_back(h16_op_d(e, l));
  for (int op : order) {
    const float m = max_of(op);
    if (m == 0.f) continue;
    if (!std::isfinite(m)) {
      r.finite = false;
      break;
    }
    if (!retune(op)) break;
  }
  // the weights (their twins for the next step when unsharded)
  const int w = h16_op_w(e);
  const float mw = max_of(w);
  if (mw != 0.f) {
    if (!std::isfinite(mw)) {
      r.finite = false;
    } else {
      const int before = e->h16_sig[w];
      retune(w);
      if (e->h16_sig[w] != before && !e->shard) refresh_from_master(e);
    }
  }
  return r;
}

void update_scales(vnt_engine* e, uint64_t batch) {
  for (uint32_t t = 0; t < ntensors(e); ++t) {
    double g;
    std::memcpy(&g, &e->h_gmax[t], sizeof g);
    if (!(g > 0.0) || !std::isfinite(g)) continue;
    const int s = kScaleTargetBits - (int)std::ceil(std::log2(g * (double)batch));
    e->scales[t] = std::clamp(s, -100, 100);
  }
}

// Adds the examples count into the exact tail (so it is summed by the collective).
__global__ void k_tail_add(long long* tail, int slot, long long v) { tail[slot] += v; }

// Examples of this round not yet in the tail (whole-node kernels add their own).
void add_examples_tail(vnt_engine* e) {
  const long long rest = (long long)e->acc_examples - (long long)e->tail_examples;
  if (rest == 0) return;
  k_tail_add<<<1, 1, 0, e->stream>>>(e->tail, kTailExamples, rest);
  VNT_LAUNCH_CHECK();
  e->launches++;
  e->tail_examples = e->acc_examples;
}

void reset_acc(vnt_engine* e) {
  e->round_open = false;
  e->acc_started = false;
  e->acc_examples = 0;
  e->acc_partials = 0;
  e->tail_examples = 0;
  e->synced = false;
}

std::vector<PassNode> local_nodes(vnt_engine* e, const uint64_t* node_sizes,
                                  const int32_t* node_device, uint32_t total_nodes,
                                  uint64_t batch_rows) {
  std::vector<PassNode> local;
  uint64_t off = 0;
  for (uint32_t n = 0; n < total_nodes; ++n) {
    if (node_sizes[n] == 0) throw EngineError(VNT_ERR_CONFIG, "virtual node with zero examples");
    const int32_t d = node_device[n];
    if (d >= (int32_t)e->devs.size())
      throw EngineError(VNT_ERR_CONFIG, "node_device references unknown local device");
    if (d >= 0) {
      if (node_sizes[n] > e->devs[d].capacity)
        throw EngineError(VNT_ERR_CAPACITY, "virtual node " + std::to_string(n) + " (" +
                                                std::to_string(node_sizes[n]) +
                                                " examples) exceeds memory capacity of device");
      local.push_back(PassNode{(int)n, d, node_sizes[n], off, 0});
    }
    off += node_sizes[n];
  }
  if (off != batch_rows)
    throw EngineError(VNT_ERR_CONFIG, "node sizes cover " + std::to_string(off) +
                                          " examples but batch has " + std::to_string(batch_rows));
  return local;
}

struct HostClock {
  vnt_engine* e;
  std::chrono::steady_clock::time_point t;
  int i = 0;
  explicit HostClock(vnt_engine* en) : e(en), t(std::chrono::steady_clock::now()) {}
  void mark() {
    if (!e->host_prof) return;
    const auto n = std::chrono::steady_clock::now();
    e->host_t[i++ & 7] += std::chrono::duration<double, std::micro>(n - t).count();
    t = n;
  }
};

int train_step_impl(vnt_engine* e, const double* x, const double* y, uint64_t batch_rows,
                    const uint64_t* node_sizes, const int32_t* node_device,
                    uint32_t total_nodes, double lr, double* loss, vnt_device_metrics* per_dev,
                    bool on_device) {
  HostClock hc(e);
  if (e->host_prof) e->host_n++;
  bind(e);
  if (!(lr > 0.0)) throw EngineError(VNT_ERR_CONFIG, "sgd_apply: learning rate must be positive");
  auto local = local_nodes(e, node_sizes, node_device, total_nodes, batch_rows);
  if (total_nodes > (1u << kMaxPartialsLog2))
    throw EngineError(VNT_ERR_CONFIG, "more than 2^21 virtual nodes: the exact int64 sum has no headroom");
  // any sum of total_nodes partials below 2^lim_bits fits int64
  e->lim_bits = std::min(kLimBits, 62 - ceil_log2(total_nodes));
  e->loss_rows = std::ldexp(1.0, ceil_log2(batch_rows));
  reset_acc(e);
  e->launches = 0;
  uint32_t retries = 0;
  const double inv_b = 1.0 / (double)batch_rows;   // virtual_exec.cpp:165
  for (int attempt = 0;; ++attempt) {
    // Device work of the step, in order; recorded once per plan as a CUDA graph.
    const Pass* graph_stage = nullptr;   // resident batch staged inside the graph
    auto enqueue_step = [&](const std::vector<StatsLaunch>* stats, bool events) {
      if (events) VNT_CUDA(cudaEventRecord(e->ev[0], e->stream));
      auto& passes = plan_for(e, local);
      if (e->node_path && passes.size() == 1) {
        step_prologue(e, passes[0], graph_stage != nullptr);   // params + zeroing + staging
      } else {
        copy_step_params(e);
        if (graph_stage) launch_stage_rows(e, *graph_stage);
        begin_round_device(e);
      }
      const bool overlap = e->comm && e->comm_overlap && !e->node_path;
      issue_pending_gathers(e);
      if (passes.size() == 1) {
        run_pass(e, passes[0], stats, true, overlap);
        e->acc_started = true;
        e->acc_examples += passes[0].examples;
      }
      add_examples_tail(e);
      if (events) VNT_CUDA(cudaEventRecord(e->ev[2], e->stream));
      if (overlap) finish_layer_collectives(e);
      else collective(e);
      if (events) VNT_CUDA(cudaEventRecord(e->ev[3], e->stream));
      launch_sgd(e);
      if (events) VNT_CUDA(cudaEventRecord(e->ev[4], e->stream));
      enqueue_readback(e, true);
    };
    bool graphed = false;
    hc.mark();   // 0: entry, local_nodes
    begin_round_host(e, batch_rows);
    fill_step_params(e, lr, inv_b);
    hc.mark();   // 1: step params
    Readback rb;
    const std::vector<Pass>* passes = local.empty() ? nullptr : &plan_for(e, local);
    const bool single = passes && passes->size() == 1;
    if (single && attempt == 0 && e->graphs && (!e->comm || e->comm->on_stream())) {
      // Graph path: host prep outside, the whole device step as one graph launch.
      const Pass& p = (*passes)[0];
      ensure_combine(e, p.nodes.size());
      ensure_capacity(e, p.rows, p.nodes.size());
      size_t off = 0;
      const std::vector<StatsLaunch> stats = prep_stats(e, p, off);
      hc.mark();   // 2: plan, capacity, stats prep
      // A device-resident batch is copied by k_stage_rows inside the graph (its
      // pointers travel in the step parameters); host batches are staged here
      // or arrive through the prefetch.
      const bool took = take_prefetch(e, x, y, local);
      const bool stage_in_graph = !took && on_device;
      if (!took && !on_device) stage_inputs(e, p, x, y, false);
      e->h_sp->x = stage_in_graph ? x : nullptr;
      e->h_sp->y = stage_in_graph ? y : nullptr;
      graph_stage = stage_in_graph ? &p : nullptr;
      hc.mark();   // 3: input staging
      // graph entry: from the memo when the mapping is the previous step's
      const bool same = e->memo.valid && e->memo.rows == batch_rows &&
                        e->memo.sizes.size() == total_nodes &&
                        std::equal(e->memo.sizes.begin(), e->memo.sizes.end(), node_sizes) &&
                        std::equal(e->memo.devs.begin(), e->memo.devs.end(), node_device);
      if (!same) {
        e->memo.sizes.assign(node_sizes, node_sizes + total_nodes);
        e->memo.devs.assign(node_device, node_device + total_nodes);
        e->memo.rows = batch_rows;
        e->memo.valid = true;
        for (auto& plane : e->memo.ge)
          for (auto& row : plane)
            for (auto& g : row) g = nullptr;
      }
      const int gathers = (e->shard && e->ag_pending) ? 1 : 0;
      vnt_engine::GraphEntry*& slot = e->memo.ge[e->cur & 1][stage_in_graph ? 1 : 0][gathers];
      if (!slot) {
        std::vector<int64_t> key = {(int64_t)e->opt.resident_rows, -1, e->cur,
                                    stage_in_graph ? 1 : 0, (int64_t)total_nodes, gathers};
        for (const auto& n : local) {
          key.push_back(n.node);
          key.push_back(n.dev);
          key.push_back((int64_t)n.rows);
          key.push_back((int64_t)n.src_row);
        }
        slot = &e->graph_cache[key];
      }
      auto& ge = *slot;
      if (ge.exec == nullptr && ge.seen == 0) {
        ge.seen = 1;   // first encounter runs eagerly (allocations, attributes)
        enqueue_step(&stats, true);
      } else {
        if (ge.exec == nullptr) {
          const uint32_t l0 = e->launches;
          const size_t p0 = e->prof_n;
          cudaGraph_t g;
          VNT_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
          try {
            enqueue_step(&stats, false);
          } catch (...) {
            cudaStreamEndCapture(e->stream, &g);
            throw;
          }
          VNT_CUDA(cudaStreamEndCapture(e->stream, &g));
          VNT_CUDA(cudaGraphInstantiate(&ge.exec, g, 0));
          cudaGraphDestroy(g);
          ge.launches = e->launches - l0;
          ge.prof_n = e->prof_n - p0;
          ge.prof_flops.assign(e->prof_flops.end() - (long)(ge.prof_n / 2), e->prof_flops.end());
        } else {
          e->acc_started = true;
          e->acc_examples = p.examples;
          if (e->shard) {   // host state the captured gathers / sharded update leave
            e->ag_pending = true;
            e->ag_wait.assign(e->L, 0);
            e->master_valid = false;
          }
          e->launches += ge.launches;
          e->prof_n = ge.prof_n;
          e->prof_flops = ge.prof_flops;
        }
        VNT_CUDA(cudaEventRecord(e->ev[0], e->stream));
        VNT_CUDA(cudaGraphLaunch(ge.exec, e->stream));
        VNT_CUDA(cudaEventRecord(e->ev[4], e->stream));
        graphed = true;
      }
      start_queued_prefetch(e);   // overlaps the next batch's H2D with this step
      hc.mark();   // 4: graph key, launch
      VNT_CUDA(cudaStreamSynchronize(e->stream));
      hc.mark();   // 5: synchronize
      rb = parse_readback(e);
    } else {
      VNT_CUDA(cudaEventRecord(e->ev[0], e->stream));
      copy_step_params(e);
      begin_round_device(e);
      // every rank issues the same collective sequence: per layer (overlapped)
      // on the layered path, one reduction otherwise
      const bool overlap = e->comm && e->comm_overlap && !e->node_path;
      if (!local.empty()) accumulate(e, local, x, y, on_device, attempt == 0, overlap);
      add_examples_tail(e);
      if (local.empty()) {
        // This process hosts no node this step: the same collectives as every
        // other rank (the weight gathers, then the reductions) with zeros.
        flush_gathers(e);
        VNT_CUDA(cudaMemsetAsync(e->G, 0, e->P * sizeof(long long), e->stream));
        if (overlap)
          for (int l = e->L - 1; l >= 0; --l) layer_collective(e, l);
      }
      VNT_CUDA(cudaEventRecord(e->ev[2], e->stream));
      if (overlap) finish_layer_collectives(e);
      else collective(e);
      VNT_CUDA(cudaEventRecord(e->ev[3], e->stream));
      launch_sgd(e);
      VNT_CUDA(cudaEventRecord(e->ev[4], e->stream));
      start_queued_prefetch(e);   // overlaps the next batch's H2D with this step
      rb = read_tail(e, true);
    }
    if (rb.nonfinite || !rb.overflow.empty() || rb.h16_range) {
      e->prof_n = 0;
      e->prof_flops.clear();
    }
    // an fp16 operand out of range (inf twins) also poisons what follows it:
    // redo at the retuned scales before judging the non-finite flag
    const H16Review h16 = h16_retune(e);
    if (rb.nonfinite && !(rb.h16_range && h16.finite)) {
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_NONFINITE, "ExactAccumulator: non-finite value");
    }
    if (!rb.overflow.empty() || rb.loss_range || rb.h16_range || h16.under) {
      if (!rb.h16_range && !h16.under) {
        for (int t : rb.overflow) e->scales[t] -= kRescaleStep;
        if (rb.loss_range) e->loss_bits -= kLossRescale;
      }
      ++retries;
      reset_acc(e);
      if (retries > 8) throw EngineError(VNT_ERR_RESCALE, "fixed-point range could not be found");
      continue;
    }
    update_scales(e, batch_rows);
    const double mean_loss = rb.loss_sum / (double)batch_rows;   // virtual_exec.cpp:275
    relax_loss_bits(e, mean_loss);
    if (loss) *loss = mean_loss;
    e->timings_graphed = graphed;
    break;
  }
  float ms[4] = {};
  if (!e->timings_graphed) {
    cudaEventElapsedTime(&ms[0], e->ev[0], e->ev[1]);
    cudaEventElapsedTime(&ms[1], e->ev[1], e->ev[2]);
    cudaEventElapsedTime(&ms[2], e->ev[2], e->ev[3]);
    cudaEventElapsedTime(&ms[3], e->ev[3], e->ev[4]);
  }
  (void)cudaGetLastError();   // timing is best-effort
  e->timings.forward_ms = ms[0];
  e->timings.backward_ms = ms[1];
  e->timings.sync_ms = ms[2];
  e->timings.update_ms = ms[3];
  cudaEventElapsedTime(&e->timings.total_ms, e->ev[0], e->ev[4]);
  (void)cudaGetLastError();
  e->timings.kernel_launches = e->launches;
  e->timings.rescale_retries = retries;
  e->timings.passes = local.empty() ? 0u : (uint32_t)plan_for(e, local).size();
  prof_collect(e);
  if (per_dev) {
    for (size_t d = 0; d < e->devs.size(); ++d) {
      vnt_device_metrics m{};
      for (const auto& pn : local) {
        if (pn.dev != (int)d) continue;
        m.waves += 1;
        m.examples += pn.rows;
        m.peak_resident = std::max<uint64_t>(m.peak_resident, pn.rows);
      }
      m.buffer_bytes = e->P * sizeof(double);
      per_dev[d] = m;
    }
  }
  reset_acc(e);
  hc.i = 6;
  hc.mark();   // 6: readback, scales, timings, metrics
  return VNT_OK;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const EngineError& err) {
    return set_error(err.code, err.what());
  } catch (const std::exception& err) {
    return set_error(VNT_ERR_INTERNAL, err.what());
  }
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

const char* vnt_last_error(void) { return g_last_error.c_str(); }

const char* vnt_build_info(void) {
  return "vnt-b200 engine: sm_100a, FFMA + tcgen05 kind::tf32, int64 exact gradient sum, NCCL";
}

int vnt_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw EngineError(VNT_ERR_NCCL, ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return VNT_OK;
  });
}

int vnt_engine_create(const vnt_model_desc* model, const vnt_engine_options* options,
                      vnt_engine** out) {
  return guarded([&] {
    if (!model || !options || !out) throw EngineError(VNT_ERR_CONFIG, "null argument");
    if (model->num_widths < 2)
      throw EngineError(VNT_ERR_CONFIG, "ModelSpec: need at least input and output widths");
    for (uint32_t i = 0; i < model->num_widths; ++i)
      if (model->layer_widths[i] == 0)
        throw EngineError(VNT_ERR_CONFIG, "ModelSpec: layer widths must be positive");
    if (model->activation < 0 || model->activation > 2 || model->loss < 0 || model->loss > 1)
      throw EngineError(VNT_ERR_CONFIG, "unknown activation or loss");
    if (options->world_size < 1 || options->rank < 0 || options->rank >= options->world_size)
      throw EngineError(VNT_ERR_CONFIG, "bad rank/world_size");
    if (options->momentum < 0.0 || options->momentum >= 1.0)
      throw EngineError(VNT_ERR_CONFIG, "momentum must lie in [0, 1)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw EngineError(VNT_ERR_CUDA, "no CUDA device visible: the B200 engine has no CPU fallback");
    if (options->cuda_device < 0 || options->cuda_device >= ndev)
      throw EngineError(VNT_ERR_CUDA, "cuda_device out of range");
    cudaDeviceProp prop;
    VNT_CUDA(cudaGetDeviceProperties(&prop, options->cuda_device));
    if (prop.major != 10)
      throw EngineError(VNT_ERR_CUDA, std::string("engine is built for sm_100a (B200); found ") +
                                          prop.name);
    auto e = std::make_unique<vnt_engine>();
    e->opt = *options;
    e->opt.nccl_id = nullptr;
    e->profile = getenv("VNT_PROFILE_KERNELS") && getenv("VNT_PROFILE_KERNELS")[0] == '1';
    e->widths.assign(model->layer_widths, model->layer_widths + model->num_widths);
    e->L = (int)model->num_widths - 1;
    e->act = model->activation;
    e->loss = model->loss;
    e->sm_count = prop.multiProcessorCount;
    uint64_t off = 0, toff = 0;
    for (int l = 0; l < e->L; ++l) {
      e->woff.push_back(off);
      off += e->widths[l] * e->widths[l + 1];
      e->boff.push_back(off);
      off += e->widths[l + 1];
      e->wtoff.push_back(toff);
      toff += e->widths[l] * e->widths[l + 1];
      e->tc_layer.push_back(tc_layer_eligible(e->opt.gemm_mode, e->widths[l], e->widths[l + 1]));
    }
    e->P = off;
    // X[0] row stride: a whole number of 128-B MN-major groups for the dW
    // operand when layer 0 runs on tcgen05 (64 fp16 / 32 fp32 features)
    const bool split_mode = e->opt.gemm_mode == VNT_GEMM_3XF16 || e->opt.gemm_mode == VNT_GEMM_AUTO;
    e->ld0 = e->tc_layer[0] ? round_up(e->widths[0], split_mode ? 64 : 32) : e->widths[0];
    {
      // Chosen from the widths alone, so every run of a model takes the same path.
      bool any_tc = false;
      uint64_t strips = 0;
      for (int l = 0; l < e->L; ++l) {
        any_tc |= e->tc_layer[l] != 0;
        strips += (e->widths[l] + 1) * ceil_div(e->widths[l + 1], (uint64_t)vntb::kNodeOC);
      }
      // CTAs per node (VNT_NODE_CLUSTER, default 4) and the rows per smem chunk
      // are fixed here, from the widths alone: the cluster size decides how a
      // node's dW rows are split and summed, so it must never depend on which
      // nodes share a pass.  The chunk bound leaves room for the
      // DSMEM exchange area at the largest chunk.
      const char* cl_env = getenv("VNT_NODE_CLUSTER");
      const int cl_req = cl_env ? atoi(cl_env) : 4;
      e->node_cl = (cl_req == 2 || cl_req == 4 || cl_req == 8) ? cl_req : 1;
      const uint64_t smem_floats = 227 * 1024 / sizeof(float) - 64;
      const uint64_t per_row = node_row_floats(e.get()), wt = node_wt_floats(e.get()) + 16;
      auto rows_fit = [&](uint64_t exchange) -> int {
        const uint64_t fixed = wt + exchange;
        return fixed >= smem_floats
                   ? 0
                   : (int)std::min<uint64_t>(256, (smem_floats - fixed) / std::max<uint64_t>(per_row, 1));
      };
      e->node_rc_max = rows_fit(e->node_cl > 1 ? strips * vntb::kNodeOC : 0);
      if (e->node_rc_max < 1 && e->node_cl > 1) {   // no room to exchange strips: one CTA per node
        e->node_cl = 1;
        e->node_rc_max = rows_fit(0);
      }
      const bool off_env = getenv("VNT_NODE_KERNEL") && getenv("VNT_NODE_KERNEL")[0] == '0';
      e->node_path = !off_env && !any_tc && e->L <= vntb::kNodeMaxLayers &&
                     strips <= (uint64_t)vntb::kNodeMaxStrips && e->node_rc_max >= 1;
    }
    bind(e.get());
    VNT_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    VNT_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    VNT_CUDA(cudaEventCreateWithFlags(&e->pf_event, cudaEventDisableTiming));
    VNT_CUDA(cudaStreamCreateWithFlags(&e->aux_stream, cudaStreamNonBlocking));
    VNT_CUDA(cudaEventCreateWithFlags(&e->fork_ev, cudaEventDisableTiming));
    VNT_CUDA(cudaEventCreateWithFlags(&e->join_ev, cudaEventDisableTiming));
    for (auto& ev : e->ev) VNT_CUDA(cudaEventCreate(&ev));
    e->w64 = (double*)dalloc(e->P * sizeof(double));
    VNT_CUDA(cudaMemset(e->w64, 0, e->P * sizeof(double)));
    if (e->opt.momentum > 0.0) {
      e->v64 = (double*)dalloc(e->P * sizeof(double));
      VNT_CUDA(cudaMemset(e->v64, 0, e->P * sizeof(double)));
    }
    e->w32 = (float*)dalloc(e->P * sizeof(float));
    VNT_CUDA(cudaMemset(e->w32, 0, e->P * sizeof(float)));
    e->wt32 = (float*)dalloc(toff * sizeof(float));
    VNT_CUDA(cudaMemset(e->wt32, 0, toff * sizeof(float)));
    e->split = split_mode;
    if (e->split) {
      e->w32h = (__half*)dalloc(e->P * sizeof(__half));
      e->w32l = (__half*)dalloc(e->P * sizeof(__half));
      // no Wᵀ twins: the forward reads W [in][out] as an MN-major operand
    }
    // split-fp16 scales before any history: activations |x| < 2^7, deltas
    // |d| < 2^5 (larger values flag kTailH16 and the step is redone at the
    // measured range); the weights' from their values (split_weights)
    e->h16_sig.assign(h16_nops(e.get()), 0);
    for (int l = 0; l <= e->L; ++l) {
      e->h16_sig[h16_op_x(e.get(), l)] = 8;
      e->h16_sig[h16_op_d(e.get(), l)] = 10;
    }
    e->ntail = kTailOverflow + ntensors(e.get());
    // zero gap after P: a sharded reduce-scatter of the last layer reads up to
    // 32 words per rank past its slice (kMaxRanks ranks)
    e->tail_off = round_up(e->P, 32) + 32 * kMaxRanks;
    const uint64_t gwords = e->tail_off + tail_words(e.get());
    e->G = (long long*)dalloc(gwords * sizeof(long long));
    VNT_CUDA(cudaMemset(e->G, 0, gwords * sizeof(long long)));
    e->tail = e->G + e->tail_off;
    e->gmax = reinterpret_cast<unsigned long long*>(e->tail + e->ntail);
    e->h16max = e->gmax + ntensors(e.get());
    e->d_word = (long long*)dalloc(8 * sizeof(long long));
    if (e->node_path) {
      e->wpad = (float*)dalloc(node_wt_floats(e.get()) * sizeof(float));
      VNT_CUDA(cudaMemset(e->wpad, 0, node_wt_floats(e.get()) * sizeof(float)));
    }
    VNT_CUDA(cudaMallocHost(&e->h_tail, tail_words(e.get()) * sizeof(long long)));
    e->h_gmax = reinterpret_cast<unsigned long long*>(e->h_tail + e->ntail);
    e->h_h16max = e->h_gmax + ntensors(e.get());
    VNT_CUDA(cudaHostGetDevicePointer((void**)&e->m_tail, e->h_tail, 0));
    e->scales.assign(ntensors(e.get()), 0);
    if (e->L > vntb::kMaxLayers) throw EngineError(VNT_ERR_CONFIG, "too many layers (max 64)");
    e->d_sp = (StepParams*)dalloc(sizeof(StepParams));
    VNT_CUDA(cudaMallocHost(&e->h_sp, sizeof(StepParams)));
    VNT_CUDA(cudaHostGetDevicePointer((void**)&e->m_sp, e->h_sp, 0));
    std::memset(e->h_sp, 0, sizeof(StepParams));
    // Events recorded inside a graph cannot be timed: profiling runs eagerly.
    e->graphs = !(getenv("VNT_GRAPHS") && getenv("VNT_GRAPHS")[0] == '0') && !e->profile;
    e->host_prof = getenv("VNT_HOST_PROFILE") && getenv("VNT_HOST_PROFILE")[0] == '1';
    tc_init(e.get());
    // VNT_FORCE_COMM=1: a one-rank NCCL group on a single process, so the
    // collective code paths (including the overlapped per-layer reduction) run
    // and can be tested on one GPU.
    const bool force = getenv("VNT_FORCE_COMM") && getenv("VNT_FORCE_COMM")[0] == '1';
    if (options->comm_ops) {
      if (options->comm_ops->size < 1 || options->comm_ops->rank < 0 ||
          options->comm_ops->rank >= options->comm_ops->size)
        throw EngineError(VNT_ERR_CONFIG, "comm_ops: bad rank/size");
      e->pool = std::make_unique<vntb::HostGroup>(*options->comm_ops);
    } else if (e->opt.world_size > 1 || force) {
      ncclUniqueId id;
      if (e->opt.world_size > 1) {
        if (!options->nccl_id) throw EngineError(VNT_ERR_CONFIG, "world_size > 1 needs nccl_id");
        std::memcpy(&id, options->nccl_id, sizeof id);
      } else {
        vntb::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
      }
      e->pool = std::make_unique<vntb::NcclGroup>(id, e->opt.rank, e->opt.world_size,
                                                  overlap_wanted() ? kCommSms : 0);
    }
    e->comm = e->pool.get();
    if (e->comm) {
      e->opt.rank = e->comm->rank();
      e->opt.world_size = e->comm->size();
    }
    e->opt.comm_ops = nullptr;
    setup_comm(e.get());
    *out = e.release();
    return VNT_OK;
  });
}

void vnt_engine_destroy(vnt_engine* e) {
  if (!e) return;
  cudaSetDevice(e->opt.cuda_device);
  cudaStreamSynchronize(e->stream);
  if (e->comm_stream) cudaStreamSynchronize(e->comm_stream);
  e->comm = nullptr;
  e->active.reset();
  e->pool.reset();
  free_shards(e);
  for (auto& ev : e->ag_ev) cudaEventDestroy(ev);
  if (e->ag_fork) cudaEventDestroy(e->ag_fork);
  if (e->d_word) cudaFree(e->d_word);
  tc_destroy(e);
  for (auto& kv : e->plans)
    for (auto& p : kv.second) cudaFree(p.d_meta);
  for (auto* p : e->scratch) cudaFree(p);
  for (void* p : {(void*)e->w32h, (void*)e->w32l})
    if (p) cudaFree(p);
  for (auto* v : {&e->Xh, &e->Xl, &e->Dh, &e->Dl})
    for (auto* p : *v)
      if (p) cudaFree(p);
  for (void* p : {(void*)e->w64, (void*)e->v64, (void*)e->w32, (void*)e->wt32, (void*)e->G,
                  (void*)e->gout, (void*)e->xbuf[0], (void*)e->ybuf[0], (void*)e->wpad,
                  (void*)e->xbuf[1], (void*)e->ybuf[1], (void*)e->logits,
                  (void*)e->vn_mean, (void*)e->vn_m2})
    if (p) cudaFree(p);
  for (auto* v : {&e->X, &e->D})
    for (auto* p : *v)
      if (p) cudaFree(p);
  for (auto* p : e->Mk)
    if (p) cudaFree(p);
  for (auto& d : e->devs) {
    cudaFree(d.mean);
    cudaFree(d.m2);
    cudaFree(d.mean_bak);
    cudaFree(d.m2_bak);
  }
  if (e->h_combine) cudaFreeHost(e->h_combine);
  if (e->h_tail) cudaFreeHost(e->h_tail);
  if (e->h_sp) cudaFreeHost(e->h_sp);
  if (e->d_sp) cudaFree(e->d_sp);
  drop_graphs(e);
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : e->prof_ev) cudaEventDestroy(ev);
  if (e->copy_stream) {
    cudaStreamSynchronize(e->copy_stream);
    cudaStreamDestroy(e->copy_stream);
  }
  if (e->pf_event) cudaEventDestroy(e->pf_event);
  if (e->host_prof && e->host_n) {
    std::fprintf(stderr, "vnt host profile (us/step over %llu steps):", (unsigned long long)e->host_n);
    for (int i = 0; i < 7; ++i) std::fprintf(stderr, " %d:%.2f", i, e->host_t[i] / (double)e->host_n);
    std::fprintf(stderr, "\n");
  }
  if (e->aux_stream) {
    cudaStreamSynchronize(e->aux_stream);
    cudaStreamDestroy(e->aux_stream);
  }
  if (e->fork_ev) cudaEventDestroy(e->fork_ev);
  if (e->comm_stream) {
    cudaStreamSynchronize(e->comm_stream);
    cudaStreamDestroy(e->comm_stream);
  }
  for (auto& ev : e->layer_ev)
    if (ev) cudaEventDestroy(ev);
  if (e->comm_ev) cudaEventDestroy(e->comm_ev);
  if (e->join_ev) cudaEventDestroy(e->join_ev);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

uint64_t vnt_engine_param_count(const vnt_engine* e) { return e ? e->P : 0; }
uint32_t vnt_engine_tensor_count(const vnt_engine* e) { return e ? ntensors(e) : 0; }

}  // extern "C"

namespace {
// fp64 master -> every fp32 copy the kernels read; a pending sharded gather
// is superseded (the master is complete on this rank).
void refresh_from_master(vnt_engine* e) {
  for (int l = 0; l < e->L; ++l) {
    const int rows = (int)e->widths[l], cols = (int)e->widths[l + 1];
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32)), block(32, 8);
    k_refresh_weight<<<grid, block, 0, e->stream>>>(e->w64 + e->woff[l], e->w32 + e->woff[l],
                                                    e->wt32 + e->wtoff[l], rows, cols);
    VNT_LAUNCH_CHECK();
    k_refresh_vec<<<(unsigned)ceil_div(cols, 256), 256, 0, e->stream>>>(
        e->w64 + e->boff[l], e->w32 + e->boff[l], (size_t)cols);
    VNT_LAUNCH_CHECK();
  }
  split_weights(e);
  e->master_valid = true;
  if (e->shard) {
    e->ag_pending = false;
    e->ag_wait.assign(e->L, 0);
    refill_ag_send(e);
  }
}
// Before the process group changes: complete master and fp32 copies on this
// rank, streams idle, graphs and the open round dropped, the old group closed.
void quiesce_for_regroup(vnt_engine* e) {
  if (e->comm) {
    gather_master(e);
    flush_gathers(e);
  }
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  if (e->comm_stream) VNT_CUDA(cudaStreamSynchronize(e->comm_stream));
  drop_graphs(e);
  reset_acc(e);
  e->comm = nullptr;
  e->active.reset();
  e->pool.reset();
  free_shards(e);
}

// Replica state from `root` of group g: fp64 master, momentum and the
// fixed-point scale history + loss quantum (numerical state).
void broadcast_replica(vnt_engine* e, vntb::CommGroup* g, int root) {
  g->broadcast(e->w64, e->P * sizeof(double), root, e->stream);
  if (e->v64) g->broadcast(e->v64, e->P * sizeof(double), root, e->stream);
  std::vector<int32_t> sc(e->scales);
  sc.insert(sc.end(), e->h16_sig.begin(), e->h16_sig.end());
  sc.push_back(e->scales_init ? 1 : 0);
  sc.push_back(e->loss_bits);
  int32_t* d_sc = (int32_t*)dalloc(sc.size() * sizeof(int32_t));
  VNT_CUDA(cudaMemcpyAsync(d_sc, sc.data(), sc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, e->stream));
  g->broadcast(d_sc, sc.size() * sizeof(int32_t), root, e->stream);
  VNT_CUDA(cudaMemcpyAsync(sc.data(), d_sc, sc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, e->stream));
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  cudaFree(d_sc);
  e->loss_bits = sc.back();
  sc.pop_back();
  e->scales_init = sc.back() != 0;
  sc.pop_back();
  e->scales.assign(sc.begin(), sc.begin() + ntensors(e));
  e->h16_sig.assign(sc.begin() + ntensors(e), sc.end());
}
}  // namespace

extern "C" {

int vnt_engine_set_params(vnt_engine* e, const double* params, uint64_t n) {
  return guarded([&] {
    if (n != e->P) throw EngineError(VNT_ERR_SHAPE, "params layout does not match model layout");
    bind(e);
    VNT_CUDA(cudaMemcpyAsync(e->w64, params, n * sizeof(double), cudaMemcpyHostToDevice, e->stream));
    if (e->v64) VNT_CUDA(cudaMemsetAsync(e->v64, 0, e->P * sizeof(double), e->stream));
    refresh_from_master(e);
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

int vnt_engine_get_params(vnt_engine* e, double* params, uint64_t n) {
  return guarded([&] {
    if (n != e->P) throw EngineError(VNT_ERR_SHAPE, "params layout does not match model layout");
    bind(e);
    gather_master(e);
    VNT_CUDA(cudaMemcpyAsync(params, e->w64, n * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

int vnt_engine_add_device(vnt_engine* e, uint64_t capacity, int32_t* out_index) {
  return guarded([&] {
    bind(e);
    vnt_engine::LDev d;
    d.capacity = capacity;
    const uint64_t in = e->widths[0];
    d.mean = (double*)dalloc(in * sizeof(double));
    d.m2 = (double*)dalloc(in * sizeof(double));
    d.mean_bak = (double*)dalloc(in * sizeof(double));
    d.m2_bak = (double*)dalloc(in * sizeof(double));
    VNT_CUDA(cudaMemset(d.mean, 0, in * sizeof(double)));
    VNT_CUDA(cudaMemset(d.m2, 0, in * sizeof(double)));
    e->devs.push_back(d);
    drop_graphs(e);
    if (out_index) *out_index = (int32_t)e->devs.size() - 1;
    return VNT_OK;
  });
}

int vnt_engine_device_count(const vnt_engine* e) { return e ? (int)e->devs.size() : 0; }
}  // extern "C"

namespace {
vnt_engine::LDev new_lineage(vnt_engine* e, uint64_t capacity) {
  vnt_engine::LDev d;
  d.capacity = capacity;
  const uint64_t in = e->widths[0];
  d.mean = (double*)dalloc(in * sizeof(double));
  d.m2 = (double*)dalloc(in * sizeof(double));
  d.mean_bak = (double*)dalloc(in * sizeof(double));
  d.m2_bak = (double*)dalloc(in * sizeof(double));
  VNT_CUDA(cudaMemset(d.mean, 0, in * sizeof(double)));
  VNT_CUDA(cudaMemset(d.m2, 0, in * sizeof(double)));
  return d;
}

void free_lineage(vnt_engine::LDev& d) {
  for (double* p : {d.mean, d.m2, d.mean_bak, d.m2_bak})
    if (p) cudaFree(p);
  d = vnt_engine::LDev{};
}

// LayerStats::combine(other) of lineage `a` with (count_b, mean_b, m2_b) on the
// device (model.cpp:123-139; the same factors and kernel as the per-node
// combine of a step, so the operation order is the reference's).
void combine_lineage(vnt_engine* e, vnt_engine::LDev& a, double count_b, const double* mean_b,
                     const double* m2_b) {
  if (count_b == 0) return;
  CombineStep st{0, 0, 0.0, 0.0};
  if (a.count == 0) {
    st.copy = 1;
    a.count = count_b;
  } else {
    const double n = a.count + count_b;
    st.f1 = a.count * count_b / n;
    st.f2 = count_b / n;
    a.count = n;
  }
  CombineStep* d_st = (CombineStep*)dalloc(sizeof st);
  VNT_CUDA(cudaMemcpyAsync(d_st, &st, sizeof st, cudaMemcpyHostToDevice, e->stream));
  const uint64_t in = e->widths[0];
  k_stats_combine<<<(unsigned)ceil_div(in, 128), 128, 0, e->stream>>>(a.mean, a.m2, (int)in, mean_b, m2_b, d_st, 1);
  VNT_LAUNCH_CHECK();
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  cudaFree(d_st);
}

// Lineage wire format over the process pool: [count | mean[in] | m2[in]] fp64.
double* lineage_packet(vnt_engine* e, uint64_t& words) {
  words = 1 + 2 * e->widths[0];
  return (double*)dalloc(words * sizeof(double));
}

void quiesce_local(vnt_engine* e) {
  VNT_CUDA(cudaStreamSynchronize(e->stream));
  if (e->aux_stream) VNT_CUDA(cudaStreamSynchronize(e->aux_stream));
  e->stats_join_pending = false;
  e->pf.valid = false;
  drop_graphs(e);
  reset_acc(e);
}
}  // namespace

extern "C" {

int vnt_engine_remap_devices(vnt_engine* e, uint32_t new_count, const int32_t* src, uint32_t n_merges,
                             const int32_t* merges) {
  return guarded([&] {
    bind(e);
    const int old = (int)e->devs.size();
    for (uint32_t k = 0; k < n_merges; ++k) {
      const int from = merges[2 * k], to = merges[2 * k + 1];
      if (from < 0 || from >= old || to < 0 || to >= old || from == to)
        throw EngineError(VNT_ERR_MIGRATION, "remap_devices: bad merge pair");
    }
    for (uint32_t i = 0; i < new_count; ++i)
      if (src[i] < -1 || src[i] >= old) throw EngineError(VNT_ERR_MIGRATION, "remap_devices: bad source");
    quiesce_local(e);
    // merges first, in order (migrate_state: removed lineages into survivors)
    for (uint32_t k = 0; k < n_merges; ++k) {
      auto& from = e->devs[merges[2 * k]];
      combine_lineage(e, e->devs[merges[2 * k + 1]], from.count, from.mean, from.m2);
    }
    // then the new list: its own lineage (a survivor), a copy of a survivor's
    // post-merge lineage (an added device), or empty (src -1)
    const uint64_t in = e->widths[0];
    std::vector<vnt_engine::LDev> next;
    for (uint32_t i = 0; i < new_count; ++i) {
      vnt_engine::LDev d = new_lineage(e, src[i] >= 0 ? e->devs[src[i]].capacity : 1);
      if (src[i] >= 0) {
        const auto& s0 = e->devs[src[i]];
        d.count = s0.count;
        VNT_CUDA(cudaMemcpyAsync(d.mean, s0.mean, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
        VNT_CUDA(cudaMemcpyAsync(d.m2, s0.m2, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
      }
      next.push_back(d);
    }
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    for (auto& d : e->devs) free_lineage(d);
    e->devs = std::move(next);
    return VNT_OK;
  });
}

int vnt_engine_send_lineage(vnt_engine* e, int32_t device, int32_t peer) {
  return guarded([&] {
    bind(e);
    if (!e->pool) throw EngineError(VNT_ERR_CONFIG, "send_lineage: the engine has no process group");
    if (device < 0 || device >= (int32_t)e->devs.size()) throw EngineError(VNT_ERR_CONFIG, "unknown device");
    quiesce_local(e);
    uint64_t words = 0;
    double* pk = lineage_packet(e, words);
    const auto& d = e->devs[device];
    const uint64_t in = e->widths[0];
    VNT_CUDA(cudaMemcpyAsync(pk, &d.count, sizeof(double), cudaMemcpyHostToDevice, e->stream));
    VNT_CUDA(cudaMemcpyAsync(pk + 1, d.mean, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
    VNT_CUDA(cudaMemcpyAsync(pk + 1 + in, d.m2, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
    log_comm(e, kLogSend, (uint64_t)peer, words);
    e->pool->send(pk, words * sizeof(double), peer, e->stream);
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    cudaFree(pk);
    return VNT_OK;
  });
}

int vnt_engine_recv_lineage(vnt_engine* e, int32_t peer, int32_t device, int32_t merge) {
  return guarded([&] {
    bind(e);
    if (!e->pool) throw EngineError(VNT_ERR_CONFIG, "recv_lineage: the engine has no process group");
    if (device < 0 || device >= (int32_t)e->devs.size()) throw EngineError(VNT_ERR_CONFIG, "unknown device");
    quiesce_local(e);
    uint64_t words = 0;
    double* pk = lineage_packet(e, words);
    log_comm(e, kLogRecv, (uint64_t)peer, words);
    e->pool->recv(pk, words * sizeof(double), peer, e->stream);
    double count = 0;
    VNT_CUDA(cudaMemcpyAsync(&count, pk, sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    const uint64_t in = e->widths[0];
    auto& d = e->devs[device];
    if (merge) {
      combine_lineage(e, d, count, pk + 1, pk + 1 + in);
    } else {   // seed: the device starts as a copy of the sender's lineage
      d.count = count;
      VNT_CUDA(cudaMemcpyAsync(d.mean, pk + 1, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
      VNT_CUDA(cudaMemcpyAsync(d.m2, pk + 1 + in, in * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
      VNT_CUDA(cudaStreamSynchronize(e->stream));
    }
    cudaFree(pk);
    return VNT_OK;
  });
}

int vnt_engine_pool_rank(const vnt_engine* e, int32_t* rank, int32_t* size) {
  if (!e) return VNT_ERR_CONFIG;
  if (rank) *rank = e->pool ? e->pool->rank() : 0;
  if (size) *size = e->pool ? e->pool->size() : 1;
  return VNT_OK;
}


int vnt_engine_device_step(vnt_engine* e, int32_t device, const double* x, const double* y,
                           const uint64_t* node_sizes, uint32_t num_nodes,
                           vnt_device_metrics* metrics) {
  return guarded([&] {
    bind(e);
    if (device < 0 || device >= (int32_t)e->devs.size())
      throw EngineError(VNT_ERR_CONFIG, "unknown device");
    if (num_nodes == 0)
      throw EngineError(VNT_ERR_CONFIG, "device_step: device has no virtual nodes to run");
    std::vector<PassNode> local;
    uint64_t off = 0;
    vnt_device_metrics m{};
    for (uint32_t k = 0; k < num_nodes; ++k) {
      if (node_sizes[k] == 0) throw EngineError(VNT_ERR_CONFIG, "Batch: count must be >= 1");
      if (node_sizes[k] > e->devs[device].capacity)
        throw EngineError(VNT_ERR_CAPACITY, "micro-batch of " + std::to_string(node_sizes[k]) +
                                                " examples exceeds memory capacity of device");
      local.push_back(PassNode{(int)k, device, node_sizes[k], off, 0});
      off += node_sizes[k];
      m.waves += 1;
      m.examples += node_sizes[k];
      m.peak_resident = std::max<uint64_t>(m.peak_resident, node_sizes[k]);
    }
    m.buffer_bytes = e->P * sizeof(double);
    if (e->synced) reset_acc(e);
    if (!e->round_open) e->launches = 0;
    // The first fixed-point scale comes from a batch estimate that every rank
    // must share (partials in different units cannot be summed): across
    // processes it is the sum of the local estimates.
    uint64_t hint = off * std::max<uint64_t>(1, e->devs.size());
    if (!e->round_open) {
      // Partials per round are counted and checked at sync (kTailPartials);
      // the loss rows bound is 2^24 examples per round.
      e->lim_bits = kLimBits;
      e->loss_rows = std::ldexp(1.0, 24);
      if (!e->scales_init && e->comm) hint = global_count(e, hint);
    }
    begin_round(e, hint);
    accumulate(e, local, x, y, false, true);
    if (metrics) *metrics = m;
    return VNT_OK;
  });
}

int vnt_engine_sync(vnt_engine* e, double* mean_grad, double* loss_sum, uint64_t* examples) {
  return guarded([&] {
    bind(e);
    if (!e->acc_started) {
      // This process accumulated nothing: contribute zeros to the collective.
      // On the first round the ranks that ran device_step agreed on the
      // initial scale with a count all-reduce; this rank takes part in it
      // with a zero count, so every rank issues the same collectives.
      uint64_t hint = 1;
      if (!e->round_open) {
        e->lim_bits = kLimBits;
        e->loss_rows = std::ldexp(1.0, 24);
        if (!e->scales_init && e->comm) hint = std::max<uint64_t>(1, global_count(e, 0));
      }
      begin_round(e, hint);
      flush_gathers(e);   // the gathers every rank with nodes issued in device_step
      VNT_CUDA(cudaMemsetAsync(e->G, 0, e->P * sizeof(long long), e->stream));
      e->acc_started = true;
    }
    add_examples_tail(e);
    if (e->acc_partials) {
      k_tail_add<<<1, 1, 0, e->stream>>>(e->tail, kTailPartials, (long long)e->acc_partials);
      VNT_LAUNCH_CHECK();
    }
    e->acc_examples = 0;
    e->tail_examples = 0;
    collective(e, true);   // the full mean gradient on every rank (sync_gradients)
    h16_reduce(e);
    Readback rb = read_tail(e, false);
    const H16Review h16 = h16_retune(e);
    if (rb.nonfinite && !(rb.h16_range && h16.finite)) {
      reset_acc(e);
      throw EngineError(VNT_ERR_NONFINITE, "ExactAccumulator: non-finite value");
    }
    if (rb.h16_range || h16.under) {
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_RESCALE, "fp16 operand range exceeded; scale lowered, redo the step");
    }
    if (rb.partials > (1ull << (62 - e->lim_bits))) {
      reset_acc(e);
      throw EngineError(VNT_ERR_CONFIG, "sync_gradients: " + std::to_string(rb.partials) +
                                            " virtual-node partials exceed the exact int64 headroom");
    }
    if (!rb.overflow.empty() || rb.loss_range) {
      for (int t : rb.overflow) e->scales[t] -= kRescaleStep;
      if (rb.loss_range) e->loss_bits -= kLossRescale;
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_RESCALE, "fixed-point range exceeded; scale lowered, redo the step");
    }
    if (rb.examples == 0) throw EngineError(VNT_ERR_CONFIG, "sync_gradients: zero examples accumulated");
    e->synced = true;
    e->timings.rescale_retries = 0;
    if (loss_sum) *loss_sum = rb.loss_sum;
    if (examples) *examples = rb.examples;
    e->h_tail[kTailExamples] = (long long)rb.examples;
    if (mean_grad) {
      if (!e->gout) e->gout = (double*)dalloc(e->P * sizeof(double));
      for (int l = 0; l < e->L; ++l) {
        for (int part = 0; part < 2; ++part) {
          const uint64_t off = part ? e->boff[l] : e->woff[l];
          const uint64_t n = part ? e->widths[l + 1] : e->widths[l] * e->widths[l + 1];
          k_mean_grad<<<(unsigned)std::min<uint64_t>(ceil_div(n, 256), 4096), 256, 0, e->stream>>>(
              e->G + off, e->gout + off, n, std::ldexp(1.0, -e->scales[2 * l + part]),
              1.0 / (double)rb.examples);
          VNT_LAUNCH_CHECK();
        }
      }
      VNT_CUDA(cudaMemcpyAsync(mean_grad, e->gout, e->P * sizeof(double), cudaMemcpyDeviceToHost,
                               e->stream));
      VNT_CUDA(cudaStreamSynchronize(e->stream));
    }
    return VNT_OK;
  });
}

int vnt_engine_take_gradient_sum(vnt_engine* e, double* sum, double* loss_sum,
                                 uint64_t* examples) {
  return guarded([&] {
    bind(e);
    if (!e->acc_started) throw EngineError(VNT_ERR_CONFIG, "no gradients accumulated");
    add_examples_tail(e);
    Readback rb = read_tail(e, false);
    const H16Review h16 = h16_retune(e);
    if (rb.nonfinite && !(rb.h16_range && h16.finite)) {
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_NONFINITE, "ExactAccumulator: non-finite value");
    }
    if (rb.h16_range || h16.under) {
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_RESCALE, "fp16 operand range exceeded; scale lowered, redo the step");
    }
    if (!rb.overflow.empty() || rb.loss_range) {
      for (int t : rb.overflow) e->scales[t] -= kRescaleStep;
      if (rb.loss_range) e->loss_bits -= kLossRescale;
      restore_stats(e);
      reset_acc(e);
      throw EngineError(VNT_ERR_RESCALE, "fixed-point range exceeded; scale lowered, redo the step");
    }
    if (!e->gout) e->gout = (double*)dalloc(e->P * sizeof(double));
    for (int l = 0; l < e->L; ++l) {
      for (int part = 0; part < 2; ++part) {
        const uint64_t off = part ? e->boff[l] : e->woff[l];
        const uint64_t n = part ? e->widths[l + 1] : e->widths[l] * e->widths[l + 1];
        // double(S) * 2^-s: exact while |S| < 2^53 (the scale keeps sums near 2^40).
        k_mean_grad<<<(unsigned)std::min<uint64_t>(ceil_div(n, 256), 4096), 256, 0, e->stream>>>(
            e->G + off, e->gout + off, n, std::ldexp(1.0, -e->scales[2 * l + part]), 1.0);
        VNT_LAUNCH_CHECK();
      }
    }
    VNT_CUDA(cudaMemcpyAsync(sum, e->gout, e->P * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    if (loss_sum) *loss_sum = rb.loss_sum;
    if (examples) *examples = rb.examples;
    reset_acc(e);
    return VNT_OK;
  });
}

int vnt_engine_set_device_capacity(vnt_engine* e, int32_t device, uint64_t capacity) {
  return guarded([&] {
    if (device < 0 || device >= (int32_t)e->devs.size())
      throw EngineError(VNT_ERR_CONFIG, "unknown device");
    e->devs[device].capacity = capacity;
    return VNT_OK;
  });
}

int vnt_engine_sgd_apply(vnt_engine* e, double lr) {
  return guarded([&] {
    bind(e);
    if (!(lr > 0.0)) throw EngineError(VNT_ERR_CONFIG, "sgd_apply: learning rate must be positive");
    if (!e->synced) throw EngineError(VNT_ERR_CONFIG, "sgd_apply: call vnt_engine_sync first");
    const uint64_t examples = (uint64_t)e->h_tail[kTailExamples];
    upload_step_params(e, lr, 1.0 / (double)examples);
    if (e->shard) load_shards_from_full(e);
    launch_sgd(e, false);   // vnt_engine_sync reduced the operand maxima
    read_tail(e, true);
    h16_retune(e);   // the weight twins this update wrote
    update_scales(e, examples);
    reset_acc(e);
    return VNT_OK;
  });
}

int vnt_engine_train_step(vnt_engine* e, const double* x, const double* y, uint64_t batch_rows,
                          const uint64_t* node_sizes, const int32_t* node_device,
                          uint32_t total_nodes, double lr, double* loss,
                          vnt_device_metrics* per_device) {
  return guarded([&] {
    return train_step_impl(e, x, y, batch_rows, node_sizes, node_device, total_nodes, lr, loss,
                           per_device, false);
  });
}

int vnt_engine_train_step_resident(vnt_engine* e, const double* x, const double* y,
                                   uint64_t batch_rows, const uint64_t* node_sizes,
                                   const int32_t* node_device, uint32_t total_nodes, double lr,
                                   double* loss, vnt_device_metrics* per_device) {
  return guarded([&] {
    return train_step_impl(e, x, y, batch_rows, node_sizes, node_device, total_nodes, lr, loss,
                           per_device, true);
  });
}

int vnt_engine_prefetch(vnt_engine* e, const double* x, const double* y, uint64_t batch_rows,
                        const uint64_t* node_sizes, const int32_t* node_device,
                        uint32_t total_nodes, int32_t x_on_device) {
  return guarded([&] {
    bind(e);
    if (e->pf.valid) {   // one batch already in flight: queue this one behind it
      auto& q = e->pf_next;
      q.x = x;
      q.y = y;
      q.rows = batch_rows;
      q.sizes.assign(node_sizes, node_sizes + total_nodes);
      q.devs.assign(node_device, node_device + total_nodes);
      q.on_device = x_on_device != 0;
      q.valid = true;
      return VNT_OK;
    }
    start_prefetch(e, x, y, batch_rows, node_sizes, node_device, total_nodes, x_on_device != 0,
                   true);
    return VNT_OK;
  });
}

int vnt_engine_get_input_stats(vnt_engine* e, int32_t device, double* count, double* mean,
                               double* m2) {
  return guarded([&] {
    bind(e);
    if (device < 0 || device >= (int32_t)e->devs.size())
      throw EngineError(VNT_ERR_CONFIG, "unknown device");
    const auto& d = e->devs[device];
    const uint64_t in = e->widths[0];
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->aux_stream));   // a statistics branch may be in flight
    if (count) *count = d.count;
    if (mean) VNT_CUDA(cudaMemcpy(mean, d.mean, in * sizeof(double), cudaMemcpyDeviceToHost));
    if (m2) VNT_CUDA(cudaMemcpy(m2, d.m2, in * sizeof(double), cudaMemcpyDeviceToHost));
    return VNT_OK;
  });
}

int vnt_engine_set_input_stats(vnt_engine* e, int32_t device, double count, const double* mean,
                               const double* m2) {
  return guarded([&] {
    bind(e);
    if (device < 0 || device >= (int32_t)e->devs.size())
      throw EngineError(VNT_ERR_CONFIG, "unknown device");
    auto& d = e->devs[device];
    const uint64_t in = e->widths[0];
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->aux_stream));
    d.count = count;
    VNT_CUDA(cudaMemcpy(d.mean, mean, in * sizeof(double), cudaMemcpyHostToDevice));
    VNT_CUDA(cudaMemcpy(d.m2, m2, in * sizeof(double), cudaMemcpyHostToDevice));
    return VNT_OK;
  });
}

uint32_t scale_count(const vnt_engine* e) {
  return ntensors(e) + (h16_reduced(e) ? (uint32_t)h16_nops(e) : 0u);
}

uint32_t vnt_engine_scale_count(const vnt_engine* e) { return e ? scale_count(e) : 0; }

int vnt_engine_get_scales(vnt_engine* e, int32_t* scales, uint32_t n) {
  return guarded([&] {
    if (n != ntensors(e) && n != scale_count(e)) throw EngineError(VNT_ERR_SHAPE, "scale count mismatch");
    std::copy(e->scales.begin(), e->scales.end(), scales);
    if (n > ntensors(e)) std::copy(e->h16_sig.begin(), e->h16_sig.end(), scales + ntensors(e));
    return VNT_OK;
  });
}

int vnt_engine_set_scales(vnt_engine* e, const int32_t* scales, uint32_t n) {
  return guarded([&] {
    if (n != ntensors(e) && n != scale_count(e)) throw EngineError(VNT_ERR_SHAPE, "scale count mismatch");
    e->scales.assign(scales, scales + ntensors(e));
    e->scales_init = true;   // explicit scales are not replaced by the first-round estimate
    if (n > ntensors(e)) {
      const bool w_changed = e->h16_sig[h16_op_w(e)] != scales[ntensors(e) + h16_op_w(e)];
      e->h16_sig.assign(scales + ntensors(e), scales + n);
      if (w_changed) {   // the weight twins follow their scale
        e->h_sp->h16_mul[h16_op_w(e)] = std::ldexp(1.f, e->h16_sig[h16_op_w(e)]);
        e->h_sp->h16_inv[h16_op_w(e)] = std::ldexp(1.f, -e->h16_sig[h16_op_w(e)]);
        copy_step_params(e);
        if (!e->shard || e->master_valid) {
          refresh_from_master(e);
        } else if (!e->ag_pending) {   // re-expand the gathered fp32 weights (ag_recv)
          e->ag_wait.assign(e->L, 1);
        }
      }
    }
    return VNT_OK;
  });
}

int vnt_engine_regroup(vnt_engine* e, int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                       int32_t source_rank) {
  return guarded([&] {
    bind(e);
    if (world_size < 1 || rank < 0 || rank >= world_size || source_rank < 0 ||
        source_rank >= world_size)
      throw EngineError(VNT_ERR_CONFIG, "bad rank/world_size/source_rank");
    quiesce_for_regroup(e);
    e->opt.rank = rank;
    e->opt.world_size = world_size;
    if (world_size > 1) {
      if (!nccl_id) throw EngineError(VNT_ERR_CONFIG, "world_size > 1 needs nccl_id");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      e->pool = std::make_unique<vntb::NcclGroup>(id, rank, world_size, overlap_wanted() ? kCommSms : 0);
      e->comm = e->pool.get();
      broadcast_replica(e, e->comm, source_rank);
    }
    setup_comm(e);
    refresh_from_master(e);
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

int vnt_engine_regroup_ops(vnt_engine* e, const vnt_comm_ops* ops, int32_t source_rank) {
  return guarded([&] {
    bind(e);
    if (!ops || ops->size < 1 || ops->rank < 0 || ops->rank >= ops->size || source_rank < 0 ||
        source_rank >= ops->size)
      throw EngineError(VNT_ERR_CONFIG, "bad comm_ops/source_rank");
    quiesce_for_regroup(e);
    e->pool = std::make_unique<vntb::HostGroup>(*ops);
    e->comm = e->pool.get();
    e->opt.rank = ops->rank;
    e->opt.world_size = ops->size;
    broadcast_replica(e, e->comm, source_rank);
    setup_comm(e);
    refresh_from_master(e);
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

int vnt_engine_set_membership(vnt_engine* e, int32_t member, int32_t source_pool_rank) {
  return guarded([&] {
    bind(e);
    if (!e->pool) throw EngineError(VNT_ERR_CONFIG, "set_membership: the engine has no process group");
    if (source_pool_rank < 0 || source_pool_rank >= e->pool->size())
      throw EngineError(VNT_ERR_CONFIG, "set_membership: bad source rank");
    // A member before the change holds a complete replica; the source must be one.
    if (e->comm) {
      gather_master(e);
      flush_gathers(e);
    }
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    if (e->comm_stream) VNT_CUDA(cudaStreamSynchronize(e->comm_stream));
    drop_graphs(e);
    reset_acc(e);
    e->comm = nullptr;
    e->active.reset();
    free_shards(e);
    std::unique_ptr<vntb::CommGroup> sub = e->pool->split(member ? 0 : -1, e->pool->rank());
    log_comm(e, kLogBroadcast, 0, e->P);
    broadcast_replica(e, e->pool.get(), source_pool_rank);
    if (member) {
      if (!sub) throw EngineError(VNT_ERR_NCCL, "set_membership: split returned no group");
      e->active = std::move(sub);
      e->comm = e->active.get();
      e->opt.rank = e->comm->rank();
      e->opt.world_size = e->comm->size();
    }
    setup_comm(e);
    refresh_from_master(e);
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

int vnt_engine_debug_activation(vnt_engine* e, int32_t layer, float* out, uint64_t rows) {
  return guarded([&] {
    bind(e);
    if (layer < 1 || layer >= e->L) throw EngineError(VNT_ERR_CONFIG, "debug_activation: hidden layers only");
    if (e->node_path) throw EngineError(VNT_ERR_CONFIG, "debug_activation: layered path only");
    if (rows > e->cap_rows) throw EngineError(VNT_ERR_CONFIG, "debug_activation: more rows than staged");
    const uint64_t w = e->widths[layer];
    uint64_t prows = 0;   // pass rows up to the last node (pad rows included)
    for (const auto& pr : e->last_rows) prows = std::max(prows, pr.first + pr.second);
    const uint64_t n = prows * w;
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    std::vector<float> pass(n);
    const bool twins_only = e->Xh[layer] && e->Mk[layer] && e->tc_layer[layer - 1];
    if (!twins_only) {
      VNT_CUDA(cudaMemcpy(pass.data(), e->X[layer], n * sizeof(float), cudaMemcpyDeviceToHost));
    } else {   // only the split-fp16 twins were written: x ~= (hi + lo) 2^-sigma (22 bits)
      std::vector<__half> hi(n), lo(n);
      VNT_CUDA(cudaMemcpy(hi.data(), e->Xh[layer], n * sizeof(__half), cudaMemcpyDeviceToHost));
      VNT_CUDA(cudaMemcpy(lo.data(), e->Xl[layer], n * sizeof(__half), cudaMemcpyDeviceToHost));
      const float inv = std::ldexp(1.f, -e->h16_sig_step[h16_op_x(e, layer)]);
      for (uint64_t i = 0; i < n; ++i) pass[i] = (__half2float(hi[i]) + __half2float(lo[i])) * inv;
    }
    // the nodes' rows in order, without the pad rows
    uint64_t r = 0;
    for (const auto& pr : e->last_rows)
      for (uint64_t k = 0; k < pr.second && r < rows; ++k, ++r)
        std::memcpy(out + r * w, pass.data() + (pr.first + k) * w, w * sizeof(float));
    return VNT_OK;
  });
}

int vnt_engine_comm_log(vnt_engine* e, uint64_t* out, uint32_t cap, uint32_t* count) {
  return guarded([&] {
    const uint32_t n = (uint32_t)(e->comm_log.size() / 3);
    if (count) *count = n;
    for (uint32_t i = 0; out && i < std::min(n, cap); ++i)
      for (int k = 0; k < 3; ++k) out[3 * i + k] = e->comm_log[3 * i + k];
    e->comm_log.clear();
    return VNT_OK;
  });
}

int vnt_engine_reset_scales(vnt_engine* e) {
  if (!e) return VNT_ERR_CONFIG;
  e->scales_init = false;
  return VNT_OK;
}

int vnt_engine_last_timings(vnt_engine* e, vnt_step_timings* out) {
  if (!e || !out) return VNT_ERR_CONFIG;
  *out = e->timings;
  return VNT_OK;
}

void* vnt_engine_stream(vnt_engine* e) { return e ? (void*)e->stream : nullptr; }

int vnt_engine_device_alloc(vnt_engine* e, uint64_t bytes, void** out) {
  return guarded([&] {
    bind(e);
    *out = dalloc(bytes);
    e->scratch.push_back(*out);
    return VNT_OK;
  });
}

int vnt_engine_device_free(vnt_engine* e, void* p) {
  return guarded([&] {
    bind(e);
    auto it = std::find(e->scratch.begin(), e->scratch.end(), p);
    if (it == e->scratch.end()) throw EngineError(VNT_ERR_CONFIG, "not an engine allocation");
    e->scratch.erase(it);
    VNT_CUDA(cudaFree(p));
    return VNT_OK;
  });
}

int vnt_engine_memcpy_h2d(vnt_engine* e, void* dst, const void* src, uint64_t bytes) {
  return guarded([&] {
    bind(e);
    VNT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, e->stream));
    VNT_CUDA(cudaStreamSynchronize(e->stream));
    return VNT_OK;
  });
}

#ifdef VNT_TC_PROBE
// Diagnostics build only: read and clear the tcgen05 GEMM barrier-wait probe
// (6 kernel kinds x {producer wait, total, MMA tempty wait, total, epilogue
// wait, total, MMA full wait, -}, summed cycles over CTAs).
int vnt_debug_tc_probe(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, vntb::tc::g_tc_probe, sizeof(vntb::tc::g_tc_probe)) != cudaSuccess)
    return 1;
  static const unsigned long long zero[6 * 16] = {};
  return cudaMemcpyToSymbol(vntb::tc::g_tc_probe, zero, sizeof(zero)) == cudaSuccess ? 0 : 1;
}
#endif

}  // extern "C"
