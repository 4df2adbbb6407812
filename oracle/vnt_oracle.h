/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Nothing on the product path
 * (paper_2009_09523_b200/, include/vnt_engine.h) may link or call this.
 *
 * Plain-C restatement of the reference `vnt` hot path (fp64, exactly rounded
 * gradient reduction) used by tests/ and bench.py (cpu_baseline "port" leg)
 * as the checker.  Pinned against the reference itself: bit-identical to
 * oracle/_ref/libvntref.so (the reference compiled from its own sources) and
 * to the reference's checked-in fig1 outputs within 1e-15
 * (tests/test_oracle.py).  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj/core). */
#ifndef VNT_ORACLE_H
#define VNT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.cpp:14-63 */
uint64_t vo_rng_key(uint64_t seed);
uint64_t vo_rng_split_label(uint64_t key, const char* label);
double vo_rng_normal(uint64_t key, uint64_t counter);

/* data.cpp:50-113 — rows [start, start+count) of the synthetic dataset (wrapping). */
int vo_synth_batch(uint64_t data_seed, uint64_t dataset_size, uint64_t in_w,
                   uint64_t out_w, uint64_t start, uint64_t count, double* x, double* y);

/* model.cpp:62-77 */
uint64_t vo_param_count(const uint64_t* widths, uint32_t nw);
/* model.cpp:170-183 */
int vo_init_params(const uint64_t* widths, uint32_t nw, uint64_t seed, double* out);

/* model.cpp:345-360 — mean gradient + mean loss over `count` rows. */
int vo_forward_backward(const uint64_t* widths, uint32_t nw, int act, int loss,
                        const double* params, const double* x, const double* y,
                        uint64_t count, double* grads, double* loss_out);

/* The same for wide models (examples in parallel, Neumaier-compensated sums
 * instead of the exact expansion: within 1-2 ulp of vo_forward_backward). */
int vo_forward_backward_wide(const uint64_t* widths, uint32_t nw, int act, int loss,
                             const double* params, const double* x, const double* y,
                             uint64_t count, double* grads, double* loss_out);
/* relu: hidden units whose |z| <= tau * max|z| (sign not resolvable in fp32)
 * take relu' from act_ext[l] (rows x w[l] activations of an fp32 run; NULL
 * entries / act_ext NULL: none); n_amb counts units whose mask was taken
 * over and differed, n_conf sign disagreements outside the band. */
int vo_forward_backward_wide_masked(const uint64_t* widths, uint32_t nw, int act, int loss,
                                    const double* params, const double* x, const double* y,
                                    uint64_t count, const float* const* act_ext, double tau,
                                    double* grads, double* loss_out, uint64_t* n_amb,
                                    uint64_t* n_conf);

/* runner.cpp:37-82 + virtual_exec.cpp:71-100,120-168,207-282: a Trainer with
 * `n_devices` devices "gpu0".."gpuN-1", uniform mapping, sequential data. */
void* vo_trainer_create(const uint64_t* widths, uint32_t nw, int act, int loss,
                        uint64_t seed, uint64_t global_batch, uint64_t virtual_nodes,
                        double lr, uint64_t data_seed, uint64_t dataset_size,
                        uint32_t n_devices);
void vo_trainer_destroy(void* h);
int vo_trainer_step(void* h, double* loss);
int vo_trainer_params(void* h, double* out, uint64_t n);
/* model.cpp:101-139 — input running stats of device `idx` (ascending id). */
int vo_trainer_input_stats(void* h, uint32_t idx, double* count, double* mean,
                           double* m2, uint64_t width);
/* elastic.cpp:106-245 restricted to uniform devices: re-deal nodes over
 * `n_devices` devices, merging removed lineages' stats into survivors and
 * seeding added devices from survivors. */
int vo_trainer_resize(void* h, uint32_t n_devices);

/* Plain SGD with momentum (no reference oracle exists for momentum — the
 * reference SGD is plain, model.cpp:364-374): v <- mu*v + g; w <- w - lr*v. */
void vo_sgd_momentum(double* w, double* v, const double* g, uint64_t n, double lr, double mu);

#ifdef __cplusplus
}
#endif
#endif
