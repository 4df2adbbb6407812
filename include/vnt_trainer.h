/* vnt_trainer.h — C-ABI over the C++ drop-in Trainer (include/vnt/runner.hpp)
 * for non-C++ callers (the Python tests / ctypes binding in INTEGRATION.md).
 * Mirrors RunnerConfig / Trainer::{step,resize,params,world}
 * (reference runner.hpp:19-69) and the host-only data/init helpers. */
#ifndef VNT_TRAINER_H
#define VNT_TRAINER_H

#include <stdint.h>

#include "vnt_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vnt_trainer vnt_trainer;

typedef struct vnt_device_spec { /* DeviceSpec, virtual_exec.hpp:25-29 */
  const char* device_id;
  const char* device_type;
  uint64_t memory_capacity;
} vnt_device_spec;

typedef struct vnt_runner_config { /* RunnerConfig, runner.hpp:19-33 */
  const uint64_t* layer_widths;
  uint32_t num_widths;
  int32_t activation;
  int32_t loss;
  uint64_t seed;
  uint64_t global_batch;
  uint64_t virtual_nodes;
  double lr;
  uint64_t data_seed;
  uint64_t dataset_size;
  int32_t shuffle_epochs;
  uint64_t shuffle_seed;
  const vnt_device_spec* devices;
  uint32_t num_devices;
  int32_t parallel_devices;
  int32_t prefetch;
  int32_t gemm_mode; /* VNT_GEMM_* */
  double momentum;
  /* B200 extensions: one process per GPU (every process passes the same
   * config; devices are placed round-robin by ascending id).  comm_ops: a
   * host-callback group; else world_size > 1 needs the 128-byte nccl_id. */
  const vnt_comm_ops* comm_ops;
  const uint8_t* nccl_id;
  int32_t rank;
  int32_t world_size;
  int32_t cuda_device;
  uint64_t resident_rows;
} vnt_runner_config;

const char* vnt_host_last_error(void);

int vnt_trainer_create(const vnt_runner_config* config, vnt_trainer** out);
void vnt_trainer_destroy(vnt_trainer* t);
uint64_t vnt_trainer_param_count(const vnt_trainer* t);
/* StepMetrics: loss and the metrics of this process's devices in ascending
 * device id (up to cap).  A process hosting no device returns loss NaN. */
int vnt_trainer_step(vnt_trainer* t, double* loss, vnt_device_metrics* per_device, uint32_t cap);
int vnt_trainer_params(vnt_trainer* t, double* out, uint64_t n);
int vnt_trainer_resize(vnt_trainer* t, const vnt_device_spec* devices, uint32_t n);
uint32_t vnt_trainer_device_count(const vnt_trainer* t);
/* Input statistics of this process's idx-th worker (ascending id): count,
 * mean[in], m2[in].  vnt_trainer_device_count: this process's workers. */
int vnt_trainer_input_stats(vnt_trainer* t, uint32_t idx, double* count, double* mean, double* m2);

/* Host-only (no GPU): SynthDataset::sequential_batch and Model::init_params. */
int vnt_synth_batch(uint64_t data_seed, uint64_t dataset_size, uint64_t in_w, uint64_t out_w,
                    uint64_t start, uint64_t count, double* x, double* y);
int vnt_init_params(const uint64_t* widths, uint32_t nw, uint64_t seed, double* out);

/* hetero::profile_device: measured B200 step times of the workload, one
 * virtual node of b rows per point (CUDA events), on cuda_device.  out_* hold
 * up to nb points (out_npts set); warnings (skipped sizes) are not returned. */
int vnt_hetero_profile_device(const uint64_t* widths, uint32_t nw, int32_t activation,
                              int32_t loss, uint64_t seed, const char* device_type,
                              uint64_t memory_capacity, const uint64_t* batch_sizes, uint32_t nb,
                              uint64_t steps, uint64_t warmup_cutoff, int32_t cuda_device,
                              int32_t gemm_mode, uint64_t* out_batch, double* out_time,
                              uint32_t* out_npts, double* out_comm);

#ifdef __cplusplus
}
#endif
#endif
