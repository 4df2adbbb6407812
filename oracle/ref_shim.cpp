// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// C-ABI shim over the *unmodified* reference `vnt` hot-path sources, compiled
// in place from /root/reference/proj/core/src by oracle/Makefile with
// -Dvnt=vntref (namespace rename so the oracle can never collide with the
// drop-in `vnt::` API).  Output: oracle/_ref/libvntref.so (git-ignored, travels
// to the GPU box with the snapshot).  Used by tests/ as the bit-exact checker
// and by bench.py's `--impl reference` / cpu_baseline legs.
//
// Every entry point wraps one reference call site:
//   vntref_trainer_*      -> Trainer (runner.hpp:38-69, runner.cpp:37-91)
//   vntref_synth_batch    -> SynthDataset::sequential_batch (data.cpp:107-113)
//   vntref_init_params    -> Model::init_params (model.cpp:170-183)
//   vntref_forward_backward -> Model::forward_backward (model.cpp:345-360)
//   vntref_accumulate_sample -> Model::accumulate_example_grads (model.cpp:238-343)
//   vntref_sync_sgd_sample   -> sync_gradients + sgd_apply (virtual_exec.cpp:146-168,
//                               model.cpp:364-374)

#include <chrono>
#include <thread>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "vnt/errors.hpp"
#include "vnt/runner.hpp"

using namespace vntref;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const CapacityError*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ShapeError*>(&e)) return 6;
  if (dynamic_cast<const ConsistencyError*>(&e)) return 7;
  if (dynamic_cast<const MigrationError*>(&e)) return 8;
  if (dynamic_cast<const InfeasibleError*>(&e)) return 5;
  if (dynamic_cast<const ProfileError*>(&e)) return 4;
  return 1;
}

ModelSpec spec_of(const uint64_t* widths, uint32_t nw, int act, int loss, uint64_t seed) {
  ModelSpec s;
  s.layer_widths.assign(widths, widths + nw);
  s.activation = act == 0 ? Activation::kRelu : act == 1 ? Activation::kTanh : Activation::kIdentity;
  s.loss = loss == 0 ? Loss::kMse : Loss::kSoftmaxCrossEntropy;
  s.seed = seed;
  return s;
}

std::vector<DeviceSpec> devices(uint32_t n, uint64_t capacity) {
  std::vector<DeviceSpec> d;
  for (uint32_t i = 0; i < n; ++i) d.push_back({"gpu" + std::to_string(i), "B200", capacity});
  return d;
}

}  // namespace

extern "C" {

const char* vntref_last_error() { return g_err.c_str(); }

void* vntref_trainer_create(const uint64_t* widths, uint32_t nw, int act, int loss,
                            uint64_t seed, uint64_t global_batch, uint64_t virtual_nodes,
                            double lr, uint64_t data_seed, uint64_t dataset_size,
                            uint32_t n_devices, uint64_t capacity, int parallel) {
  try {
    RunnerConfig c;
    c.model = spec_of(widths, nw, act, loss, seed);
    c.global_batch = global_batch;
    c.virtual_nodes = virtual_nodes;
    c.lr = lr;
    c.data_seed = data_seed;
    c.dataset_size = dataset_size;
    c.devices = devices(n_devices, capacity);
    c.parallel_devices = parallel != 0;
    return new Trainer(c);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// Same, with the data-order options (runner.hpp:28-30): shuffled epochs and
// the background prefetch future.
void* vntref_trainer_create_ex(const uint64_t* widths, uint32_t nw, int act, int loss,
                               uint64_t seed, uint64_t global_batch, uint64_t virtual_nodes,
                               double lr, uint64_t data_seed, uint64_t dataset_size,
                               uint32_t n_devices, uint64_t capacity, int parallel,
                               int shuffle_epochs, uint64_t shuffle_seed, int prefetch) {
  try {
    RunnerConfig c;
    c.model = spec_of(widths, nw, act, loss, seed);
    c.global_batch = global_batch;
    c.virtual_nodes = virtual_nodes;
    c.lr = lr;
    c.data_seed = data_seed;
    c.dataset_size = dataset_size;
    c.devices = devices(n_devices, capacity);
    c.parallel_devices = parallel != 0;
    c.shuffle_epochs = shuffle_epochs != 0;
    c.shuffle_seed = shuffle_seed;
    c.prefetch = prefetch != 0;
    return new Trainer(c);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void vntref_trainer_destroy(void* h) { delete static_cast<Trainer*>(h); }

int vntref_trainer_step(void* h, double* loss) {
  try {
    const StepMetrics m = static_cast<Trainer*>(h)->step();
    if (loss) *loss = m.loss;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

uint64_t vntref_trainer_param_count(void* h) {
  return static_cast<Trainer*>(h)->params().values.size();
}

int vntref_trainer_params(void* h, double* out, uint64_t n) {
  const auto& v = static_cast<Trainer*>(h)->params().values;
  if (n != v.size()) return 6;
  std::memcpy(out, v.data(), n * sizeof(double));
  return 0;
}

int vntref_trainer_resize(void* h, uint32_t n_devices, uint64_t capacity) {
  try {
    static_cast<Trainer*>(h)->resize(devices(n_devices, capacity));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Input running statistics of worker `idx` (World order = ascending device id).
int vntref_trainer_input_stats(void* h, uint32_t idx, double* count, double* mean,
                               double* m2, uint64_t width) {
  const auto& w = static_cast<Trainer*>(h)->world().workers.at(idx);
  const auto it = w.kernels.layers.find("input");
  if (it == w.kernels.layers.end()) {
    *count = 0;
    return 0;
  }
  *count = it->second.count;
  if (it->second.mean.size() != width) return 6;
  std::memcpy(mean, it->second.mean.data(), width * sizeof(double));
  std::memcpy(m2, it->second.m2.data(), width * sizeof(double));
  return 0;
}

int vntref_synth_batch(uint64_t data_seed, uint64_t dataset_size, uint64_t in_w,
                       uint64_t out_w, uint64_t start, uint64_t count, double* x,
                       double* y) {
  try {
    SynthDataset d(data_seed, dataset_size, in_w, out_w);
    const Batch b = d.sequential_batch(start, count);
    std::memcpy(x, b.examples.data(), b.examples.size() * sizeof(double));
    std::memcpy(y, b.labels.data(), b.labels.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int vntref_init_params(const uint64_t* widths, uint32_t nw, int act, int loss,
                       uint64_t seed, double* out) {
  try {
    Model m(spec_of(widths, nw, act, loss, seed));
    const ParamVector p = m.init_params();
    std::memcpy(out, p.values.data(), p.values.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Mean gradient and mean loss of `count` rows at `params` (the full-batch oracle
// used by test_virtual_exec.cpp:184-201).
int vntref_forward_backward(const uint64_t* widths, uint32_t nw, int act, int loss,
                            const double* params, const double* x, const double* y,
                            uint64_t count, double* grads, double* loss_out) {
  try {
    Model m(spec_of(widths, nw, act, loss, 0));
    ParamVector p{m.layout(), std::vector<double>(params, params + m.param_count())};
    Batch b;
    b.count = count;
    b.input_width = widths[0];
    b.output_width = widths[nw - 1];
    b.examples.assign(x, x + count * widths[0]);
    b.labels.assign(y, y + count * widths[nw - 1]);
    b.ids.resize(count);
    for (uint64_t i = 0; i < count; ++i) b.ids[i] = i;
    const auto r = m.forward_backward(p, b, m.init_kernels());
    std::memcpy(grads, r.grads.values.data(), r.grads.values.size() * sizeof(double));
    *loss_out = r.loss;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Bounded CPU sample for wide models: per-example forward/backward + exact
// accumulation of `count` rows (one GradientBuffer's worth of work), then one
// rounding.  Returns seconds spent in accumulate_example_grads and in rounded().
int vntref_accumulate_sample(const uint64_t* widths, uint32_t nw, int act, int loss,
                             uint64_t seed, const double* x, const double* y,
                             uint64_t count, double* accumulate_s, double* round_s) {
  try {
    Model m(spec_of(widths, nw, act, loss, seed));
    const ParamVector p = m.init_params();
    Batch b;
    b.count = count;
    b.input_width = widths[0];
    b.output_width = widths[nw - 1];
    b.examples.assign(x, x + count * widths[0]);
    b.labels.assign(y, y + count * widths[nw - 1]);
    b.ids.resize(count);
    for (uint64_t i = 0; i < count; ++i) b.ids[i] = i;
    ExactVectorAccumulator acc(m.param_count());
    ExactAccumulator loss_sum;
    auto t0 = std::chrono::steady_clock::now();
    m.accumulate_example_grads(p, b, acc, loss_sum);
    auto t1 = std::chrono::steady_clock::now();
    volatile double sink = acc.rounded()[0];
    (void)sink;
    auto t2 = std::chrono::steady_clock::now();
    *accumulate_s = std::chrono::duration<double>(t1 - t0).count();
    *round_s = std::chrono::duration<double>(t2 - t1).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Multi-threaded bounded sample: `threads` workers, each with its own exact
// accumulator (as each simulated device has its own GradientBuffer), each
// accumulating `per_thread` examples.  Returns the wall time of the parallel
// accumulate phase (examples / wall = throughput on this many host cores).
int vntref_accumulate_sample_mt(const uint64_t* widths, uint32_t nw, int act, int loss,
                                uint64_t seed, const double* x, const double* y,
                                uint64_t per_thread, uint32_t threads, double* wall_s) {
  try {
    Model m(spec_of(widths, nw, act, loss, seed));
    const ParamVector p = m.init_params();
    std::vector<std::unique_ptr<ExactVectorAccumulator>> accs;
    for (uint32_t t = 0; t < threads; ++t)
      accs.push_back(std::make_unique<ExactVectorAccumulator>(m.param_count()));
    Batch b;
    b.count = per_thread;
    b.input_width = widths[0];
    b.output_width = widths[nw - 1];
    b.examples.assign(x, x + per_thread * widths[0]);
    b.labels.assign(y, y + per_thread * widths[nw - 1]);
    b.ids.resize(per_thread);
    for (uint64_t i = 0; i < per_thread; ++i) b.ids[i] = i;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        ExactAccumulator ls;
        m.accumulate_example_grads(p, b, *accs[t], ls);
      });
    for (auto& th : pool) th.join();
    *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}


}  // extern "C"
