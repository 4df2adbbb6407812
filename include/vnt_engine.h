/* vnt_engine.h — the thin C-ABI between the reference-compatible C++ host
 * layer (include/vnt/ headers, the `vnt::` drop-in) and the B200 CUDA engine
 * (paper_2009_09523_b200/csrc/).  Plain pointers and sizes only; all CUDA /
 * NCCL state lives behind the opaque `vnt_engine`.  There is no CPU fallback:
 * every compute entry point fails with VNT_ERR_CUDA when no sm_100 device is
 * usable.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to /root/reference/proj/core):
 *
 *   vnt_engine_create        Model::Model + make_world          model.hpp:98-106, virtual_exec.cpp:194-205
 *   vnt_engine_set_params    World replica assignment / init    model.cpp:170-183
 *   vnt_engine_add_device    WorkerState{DeviceSpec,...}        virtual_exec.hpp:100-104
 *   vnt_engine_device_step   device_step                        virtual_exec.hpp:89-92, .cpp:120-144
 *   vnt_engine_sync          sync_gradients                     virtual_exec.hpp:97-98, .cpp:146-168
 *   vnt_engine_sgd_apply     sgd_apply on every replica         model.hpp:130, model.cpp:364-374
 *   vnt_engine_train_step    train_step                         virtual_exec.hpp:130-132, .cpp:207-282
 *   vnt_engine_{get,set}_input_stats  StatefulKernelState       model.hpp:65-93, elastic.cpp:50-88
 *
 * Numerical contract: per-virtual-node fp32 gradients are
 * quantised to int64 fixed point (power-of-two scale per tensor) and summed
 * exactly, so the reduced gradient — and the whole trajectory — is a function
 * of the virtual-node partition only, never of the device mapping or count.
 */
#ifndef VNT_ENGINE_H
#define VNT_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference exception classes (errors.hpp:13-58);
 * the CLI exit-code mapping is vnt.cpp:395-413. */
#define VNT_OK 0
#define VNT_ERR_INTERNAL 1        /* vnt::Error (generic)                */
#define VNT_ERR_CONFIG 2          /* vnt::ConfigError                    */
#define VNT_ERR_CAPACITY 3        /* vnt::CapacityError                  */
#define VNT_ERR_PROFILE 4         /* vnt::ProfileError (hetero)          */
#define VNT_ERR_INFEASIBLE 5      /* vnt::InfeasibleError (hetero solve) */
#define VNT_ERR_SHAPE 6           /* vnt::ShapeError                     */
#define VNT_ERR_CONSISTENCY 7     /* vnt::ConsistencyError               */
#define VNT_ERR_MIGRATION 8       /* vnt::MigrationError                 */
#define VNT_ERR_CUDA 9            /* no usable sm_100 GPU / CUDA failure */
#define VNT_ERR_NCCL 10           /* collective failure                  */
#define VNT_ERR_NONFINITE 11      /* non-finite gradient (exact_sum.cpp:17-19) */
#define VNT_ERR_RESCALE 12        /* fixed-point range exceeded; scale lowered, redo the step */

/* model.hpp:20-21 enum order */
#define VNT_ACT_RELU 0
#define VNT_ACT_TANH 1
#define VNT_ACT_IDENTITY 2
#define VNT_LOSS_MSE 0
#define VNT_LOSS_SOFTMAX_CE 1

/* GEMM arithmetic for the dense layers.  Selection depends on layer widths
 * only (never on rows), so it is identical on every rank. */
#define VNT_GEMM_AUTO 0        /* = VNT_GEMM_3XF16 for wide layers, FFMA fp32 otherwise     */
#define VNT_GEMM_FFMA 1        /* fp32 FFMA everywhere (exact fp32 products)          */
#define VNT_GEMM_TF32 2        /* tcgen05 kind::tf32, 1 pass                         */
#define VNT_GEMM_3XF16 3       /* tcgen05 kind::f16 on split-fp16 operands             */
                               /* (x 2^s = hi + lo, hi*hi + hi*lo + lo*hi, 22 bits)     */
#define VNT_GEMM_3XTF32 VNT_GEMM_3XF16   /* round-1 name of the split mode           */

typedef struct vnt_engine vnt_engine;

/* Host-callback process group (emulation / testing backend).  The product
 * path is NCCL (vnt_engine_options::nccl_id); with comm_ops set instead, every
 * collective of the engine is carried out by these callbacks on pinned HOST
 * buffers after the engine synchronised its stream — e.g. several processes or
 * threads sharing one GPU, exchanging through gloo or shared memory.  Every
 * callback returns 0 on success; all members call collectives in the same
 * order (as NCCL requires). */
#define VNT_COMM_SUM_I64 0   /* allreduce op: int64 sum                    */
#define VNT_COMM_MAX_U64 1   /* allreduce op: uint64 max                   */
typedef struct vnt_comm_ops {
  void* ctx;
  int32_t rank;
  int32_t size;
  int (*allreduce)(void* ctx, void* buf, uint64_t count, int32_t op);
  /* recv[recv_count] = this rank's block of the int64 sum of send[size * recv_count] */
  int (*reduce_scatter)(void* ctx, const void* send, void* recv, uint64_t recv_count);
  /* recv[size * bytes] = concatenation over ranks of send[bytes] */
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
  int (*broadcast)(void* ctx, void* buf, uint64_t bytes, int32_t root);
  int (*send)(void* ctx, const void* buf, uint64_t bytes, int32_t peer);
  int (*recv)(void* ctx, void* buf, uint64_t bytes, int32_t peer);
  /* Collective: members with color >= 0 form a sub-group ranked by key; fills
   * *out (out->ctx = NULL for non-members). */
  int (*split)(void* ctx, int32_t color, int32_t key, struct vnt_comm_ops* out);
  void (*release)(void* ctx);  /* nullable: called when the engine drops the group */
} vnt_comm_ops;

typedef struct vnt_model_desc {
  const uint64_t* layer_widths; /* ModelSpec::layer_widths (model.hpp:27-37) */
  uint32_t num_widths;
  int32_t activation;           /* VNT_ACT_*  */
  int32_t loss;                 /* VNT_LOSS_* */
} vnt_model_desc;

typedef struct vnt_engine_options {
  int32_t cuda_device;     /* CUDA ordinal driven by this process                  */
  int32_t rank;            /* NCCL rank of this process                            */
  int32_t world_size;      /* processes in the NCCL group (1: no collective)       */
  const uint8_t* nccl_id;  /* 128-byte ncclUniqueId from rank 0, NULL if world 1   */
  int32_t gemm_mode;       /* VNT_GEMM_*                                           */
  double momentum;         /* 0: plain SGD exactly as the reference                */
  uint64_t resident_rows;  /* rows resident per pass (0: what 85 % of free HBM holds) */
  const vnt_comm_ops* comm_ops; /* host-callback group instead of NCCL (NULL: NCCL) */
} vnt_engine_options;

typedef struct vnt_device_metrics { /* DeviceStepMetrics, virtual_exec.hpp:72-78 */
  uint64_t waves;
  uint64_t examples;
  uint64_t peak_resident;
  uint64_t buffer_bytes;   /* modeled: 8 * |params| (acceptance criterion 10) */
} vnt_device_metrics;

typedef struct vnt_step_timings { /* device time of the last train step, ms (CUDA events) */
  float total_ms;
  float forward_ms;
  float backward_ms;
  float sync_ms;
  float update_ms;
  uint32_t kernel_launches;
  uint32_t rescale_retries;
  /* Dense-layer GEMM launches only, filled when VNT_PROFILE_KERNELS=1 (events
   * around each launch on the engine stream): summed device time, algorithmic
   * flops (2*M*N*K per launch) and launch count. */
  float gemm_ms;
  uint32_t gemm_launches;
  double gemm_flops;
  uint32_t passes;         /* passes of resident nodes the step ran (this process) */
} vnt_step_timings;

const char* vnt_last_error(void);
const char* vnt_build_info(void);

/* 128-byte NCCL unique id for vnt_engine_options::nccl_id (rank 0 creates it). */
int vnt_nccl_unique_id(uint8_t out[128]);

int vnt_engine_create(const vnt_model_desc* model, const vnt_engine_options* options,
                      vnt_engine** out);
void vnt_engine_destroy(vnt_engine* e);
uint64_t vnt_engine_param_count(const vnt_engine* e);

/* Replica parameters, reference layout (model.cpp:62-77), fp64 master copy. */
int vnt_engine_set_params(vnt_engine* e, const double* params, uint64_t n);
int vnt_engine_get_params(vnt_engine* e, double* params, uint64_t n);

/* Adds a logical device (a World worker) hosted by this process. */
int vnt_engine_add_device(vnt_engine* e, uint64_t memory_capacity, int32_t* out_index);
int vnt_engine_device_count(const vnt_engine* e);

/* device_step: the device's node micro-batches, ascending node id, rows
 * concatenated (x: rows x in, y: rows x out, fp64 host).  Accumulates the
 * example-weighted gradient sum into the process gradient buffer and updates
 * the device's input statistics. */
int vnt_engine_device_step(vnt_engine* e, int32_t device, const double* x, const double* y,
                           const uint64_t* node_sizes, uint32_t num_nodes,
                           vnt_device_metrics* metrics);

/* sync_gradients: exact sum of every device buffer (and, world_size > 1, every
 * process) divided by the examples accumulated.  mean_grad (nullable, P
 * doubles) receives the reduced mean; loss_sum receives the exact loss sum. */
int vnt_engine_sync(vnt_engine* e, double* mean_grad, double* loss_sum,
                    uint64_t* examples);

/* The process-local example-summed gradient (no collective), as the
 * reference GradientBuffer::rounded_sum() of one device (virtual_exec.cpp:
 * 102-118): sum[P] = double(S) * 2^-s per tensor, exact while |S| < 2^53.
 * Closes the accumulation round. */
int vnt_engine_take_gradient_sum(vnt_engine* e, double* sum, double* loss_sum,
                                 uint64_t* examples);
int vnt_engine_set_device_capacity(vnt_engine* e, int32_t device, uint64_t capacity);

/* sgd_apply with the synced gradient on this replica (plus momentum if set). */
int vnt_engine_sgd_apply(vnt_engine* e, double lr);

/* train_step: the whole global batch (x: batch_rows x in, y: batch_rows x out,
 * fp64 host).  node_sizes[total_nodes] partitions the rows contiguously by node
 * id; node_device[n] is the local device index running node n, or -1 if node n
 * runs in another process.  per_device (nullable) receives one entry per local
 * device. */
int vnt_engine_train_step(vnt_engine* e, const double* x, const double* y,
                          uint64_t batch_rows, const uint64_t* node_sizes,
                          const int32_t* node_device, uint32_t total_nodes, double lr,
                          double* loss, vnt_device_metrics* per_device);

/* Same, with the fp64 batch already resident in device memory (bench `value`). */
int vnt_engine_train_step_resident(vnt_engine* e, const double* x_dev, const double* y_dev,
                                   uint64_t batch_rows, const uint64_t* node_sizes,
                                   const int32_t* node_device, uint32_t total_nodes,
                                   double lr, double* loss, vnt_device_metrics* per_device);

/* Prefetch (runner.cpp:64-73 on the device): stage the rows this process
 * needs from a future step's batch on a copy stream, into the spare input
 * buffer.  One batch is in flight at a time: called while none is, the copy
 * starts now; otherwise the request is queued and the next train_step starts
 * it right after launching its own work, so the H2D overlaps that step's
 * compute.  A train_step with the same (x, y) pointers consumes the staged
 * batch and skips its own copy; any other step discards it.  The caller keeps
 * (x, y) unchanged until that step.  Multi-pass plans ignore prefetch. */
int vnt_engine_prefetch(vnt_engine* e, const double* x, const double* y, uint64_t batch_rows,
                        const uint64_t* node_sizes, const int32_t* node_device,
                        uint32_t total_nodes, int32_t x_on_device);

/* LayerStats "input" of a local device (model.hpp:65-76): count, mean[in], m2[in]. */
int vnt_engine_get_input_stats(vnt_engine* e, int32_t device, double* count, double* mean,
                               double* m2);
int vnt_engine_set_input_stats(vnt_engine* e, int32_t device, double count,
                               const double* mean, const double* m2);

/* Scale state (part of the numerical state: migrated on resize).  n =
 * vnt_engine_tensor_count: the fixed-point scales 2^s per gradient tensor;
 * n = vnt_engine_scale_count: followed by the split-fp16 operand exponents
 * sigma (VNT_GEMM_3XF16), the full state a bitwise-continued trajectory
 * needs.  Scales set here are authoritative: the first round does not
 * replace them with its batch-size estimate. */
int vnt_engine_get_scales(vnt_engine* e, int32_t* scales, uint32_t n);
int vnt_engine_set_scales(vnt_engine* e, const int32_t* scales, uint32_t n);
uint32_t vnt_engine_tensor_count(const vnt_engine* e);
uint32_t vnt_engine_scale_count(const vnt_engine* e);
/* Elastic resize across processes (elastic.cpp:106-245 at the process level):
 * join a new NCCL group (world_size, rank, 128-byte id from its rank 0) and
 * take the replica state — fp64 parameters, momentum and the fixed-point
 * scale history — from `source_rank` by broadcast.  Per-device input
 * statistics migrate through vnt_engine_{get,set}_input_stats (the host
 * layer applies migrate_state's merge/seed rules).  world_size 1 leaves the
 * group and keeps the local state. */
int vnt_engine_regroup(vnt_engine* e, int32_t rank, int32_t world_size, const uint8_t* nccl_id,
                       int32_t source_rank);

/* Same with a host-callback group (vnt_comm_ops) as the new process group. */
int vnt_engine_regroup_ops(vnt_engine* e, const vnt_comm_ops* ops, int32_t source_rank);
/* Elastic resize within the job's process pool (the group the engine was
 * created with): collective over the pool.  Processes passing member != 0
 * form the group that trains from now on (ranked by pool rank); the others
 * stay idle until a later call makes them members again.  Every process
 * receives the replica state — fp64 parameters, momentum, scale history —
 * from pool rank source_pool_rank (a member of the previous training group). */
int vnt_engine_set_membership(vnt_engine* e, int32_t member, int32_t source_pool_rank);

/* Elastic resize of this process's logical devices (elastic.cpp:106-245 on
 * the GPU): first the merges, in order — merges[2k] (old index, a removed
 * lineage) is combined into merges[2k+1] (old index, a survivor) as
 * LayerStats::combine (model.cpp:123-139); then new device i takes old
 * lineage src[i] (a survivor's own, or a copy of a survivor's post-merge
 * lineage for an added device; -1: empty).  Capacities are set afterwards
 * with vnt_engine_set_device_capacity. */
int vnt_engine_remap_devices(vnt_engine* e, uint32_t new_count, const int32_t* src,
                             uint32_t n_merges, const int32_t* merges);
/* Cross-process lineage moves over the process pool (a removed device's
 * statistics to its survivor, a survivor's to an added device): the sender
 * ships (count, mean, m2) of its local device; the receiver combines it into
 * (merge != 0) or overwrites (seed) its local device.  Pairs must be issued
 * in the same order on every process. */
int vnt_engine_send_lineage(vnt_engine* e, int32_t device, int32_t peer);
int vnt_engine_recv_lineage(vnt_engine* e, int32_t peer, int32_t device, int32_t merge);
/* This process's rank / size in the process pool (0 / 1 without a group). */
int vnt_engine_pool_rank(const vnt_engine* e, int32_t* rank, int32_t* size);

/* Forget the scale history: the next step uses the deterministic initial scale
 * 40 - ceil(log2 B) (stateless callers, e.g. vnt::train_step on a World). */
int vnt_engine_reset_scales(vnt_engine* e);

int vnt_engine_last_timings(vnt_engine* e, vnt_step_timings* out);
/* Diagnostics: the collectives issued since the last call, as (op, offset,
 * count) triples in issue order (up to cap triples copied, *count = triples
 * logged).  op: 1 all-reduce (int64 sum), 2 reduce-scatter, 3 all-gather,
 * 4 max all-reduce, 5 count agreement, 6 replica broadcast, 7 send, 8 recv;
 * offset = position in the parameter layout (gradient buffer words).  Every
 * rank of a group must issue the identical sequence; clears the log. */
int vnt_engine_comm_log(vnt_engine* e, uint64_t* out, uint32_t cap, uint32_t* count);
/* Diagnostics (tests): hidden activations X[layer] (rows x width, fp32) of
 * the last pass, its nodes' rows in order (pad rows dropped), e.g. to resolve
 * relu masks at near-zero pre-activations when comparing with an fp64
 * reference; (hi + lo) 2^-sigma when only split-fp16 twins exist.  Layered
 * path only. */
int vnt_engine_debug_activation(vnt_engine* e, int32_t layer, float* out, uint64_t rows);
/* The CUDA stream the engine launches on (cudaStream_t as void*). */
void* vnt_engine_stream(vnt_engine* e);
/* Scratch device allocation owned by the engine (bench/test staging). */
int vnt_engine_device_alloc(vnt_engine* e, uint64_t bytes, void** out);
int vnt_engine_device_free(vnt_engine* e, void* p);
int vnt_engine_memcpy_h2d(vnt_engine* e, void* dst, const void* src, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* VNT_ENGINE_H */
