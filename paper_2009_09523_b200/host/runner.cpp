// vnt drop-in: Trainer (reference runner.cpp semantics) over a persistent
// B200 engine: parameters stay in HBM, the batch of each step is the same
// function of (data_seed, shuffle_seed, step) as in the reference.
#include "vnt/runner.hpp"

#include <algorithm>
#include <map>

#include "gpu_model.hpp"
#include "vnt/errors.hpp"
#include "vnt/rng.hpp"
#include "vnt_engine.h"

namespace vnt {

void RunnerConfig::validate() const {
  model.validate();
  if (global_batch == 0) throw ConfigError("RunnerConfig: global batch must be >= 1");
  if (virtual_nodes == 0) throw ConfigError("RunnerConfig: need at least one virtual node");
  if (global_batch % virtual_nodes != 0)
    throw ConfigError("RunnerConfig: virtual node count must divide the global batch");
  if (!(lr > 0)) throw ConfigError("RunnerConfig: learning rate must be positive");
  if (devices.empty()) throw ConfigError("RunnerConfig: device list is empty");
  const std::size_t n = dataset_size == 0 ? global_batch : dataset_size;
  if (n < global_batch) throw ConfigError("RunnerConfig: dataset smaller than one batch");
  if (shuffle_epochs && n % global_batch != 0)
    throw ConfigError("RunnerConfig: shuffled epochs need batch-aligned dataset size");
  if (momentum < 0.0 || momentum >= 1.0) throw ConfigError("RunnerConfig: momentum must lie in [0, 1)");
}

namespace {
RunnerConfig checked(RunnerConfig c) {
  c.validate();
  return c;
}

std::vector<DeviceSpec> sorted_devices(std::vector<DeviceSpec> d) {
  std::sort(d.begin(), d.end(), [](const DeviceSpec& a, const DeviceSpec& b) { return a.device_id < b.device_id; });
  return d;
}
}  // namespace

Trainer::Trainer(RunnerConfig config)
    : config_(checked(std::move(config))),
      model_(config_.model),
      data_(config_.data_seed, config_.dataset_size ? config_.dataset_size : config_.global_batch,
            config_.model.layer_widths.front(), config_.model.layer_widths.back()),
      mapping_(make_uniform_mapping(config_.global_batch, config_.virtual_nodes, config_.devices)),
      world_devices_(sorted_devices(config_.devices)) {
  std::vector<std::uint64_t> w(config_.model.layer_widths.begin(), config_.model.layer_widths.end());
  const vnt_model_desc d{w.data(), (uint32_t)w.size(), (int32_t)config_.model.activation,
                         (int32_t)config_.model.loss};
  vnt_engine_options o{};
  o.cuda_device = config_.cuda_device;
  o.world_size = 1;
  o.gemm_mode = config_.gemm_mode ? config_.gemm_mode : detail::engine_gemm_mode();
  o.momentum = config_.momentum;
  raise_status(vnt_engine_create(&d, &o, &engine_), "Trainer");
  const ParamVector p = model_.init_params();
  raise_status(vnt_engine_set_params(engine_, p.values.data(), p.values.size()), "Trainer");
  bind_devices();
}

Trainer::~Trainer() { vnt_engine_destroy(engine_); }

// Engine logical device i == world_devices_[i] (ascending id, World order).
void Trainer::bind_devices() {
  while (vnt_engine_device_count(engine_) < (int)world_devices_.size()) {
    int32_t idx;
    raise_status(vnt_engine_add_device(engine_, 1, &idx), "Trainer");
  }
  for (std::size_t i = 0; i < world_devices_.size(); ++i)
    raise_status(vnt_engine_set_device_capacity(engine_, (int32_t)i, world_devices_[i].memory_capacity),
                 "Trainer");
}

Batch Trainer::batch_for_step(std::uint64_t step) {
  const std::size_t n = data_.size();
  const std::uint64_t start = (step * config_.global_batch) % n;
  if (!config_.shuffle_epochs) return data_.sequential_batch(start, config_.global_batch);
  const std::uint64_t epoch = step * config_.global_batch / n;
  if (perm_epoch_ != epoch) {
    perm_ = random_permutation(CounterRng(config_.shuffle_seed).split("epoch").split(epoch), n);
    perm_epoch_ = epoch;
  }
  std::vector<std::uint64_t> ids(perm_.begin() + start, perm_.begin() + start + config_.global_batch);
  return data_.batch(ids);
}

Batch Trainer::next_batch() {
  if (!config_.prefetch) return batch_for_step(step_);
  Batch b = (prefetched_ && prefetched_step_ == step_) ? prefetched_->get() : batch_for_step(step_);
  prefetched_step_ = step_ + 1;
  prefetched_ = std::async(std::launch::async, [this, s = step_ + 1] { return batch_for_step(s); });
  return b;
}

StepMetrics Trainer::step() {
  const Batch batch = next_batch();
  std::map<std::string, int> index;
  for (std::size_t i = 0; i < world_devices_.size(); ++i) index[world_devices_[i].device_id] = (int)i;
  std::vector<int32_t> node_dev(mapping_.total_nodes(), -1);
  for (const auto& [dev, nodes] : mapping_.assignments)
    for (auto n : nodes) node_dev[n] = index.at(dev);
  std::vector<std::uint64_t> sizes(mapping_.node_sizes.begin(), mapping_.node_sizes.end());
  std::vector<vnt_device_metrics> dm(std::max(world_devices_.size(),
                                              (std::size_t)vnt_engine_device_count(engine_)));
  double loss = 0;
  raise_status(vnt_engine_train_step(engine_, batch.examples.data(), batch.labels.data(), batch.count,
                                     sizes.data(), node_dev.data(), (uint32_t)sizes.size(), config_.lr,
                                     &loss, dm.data()),
               "Trainer::step");
  params_cache_.reset();
  world_cache_.reset();
  StepMetrics m;
  m.step = step_;
  m.loss = loss;
  for (std::size_t i = 0; i < world_devices_.size(); ++i)
    m.per_device.push_back({world_devices_[i].device_id, dm[i].waves, dm[i].examples,
                            dm[i].peak_resident, dm[i].buffer_bytes});
  ++step_;
  return m;
}

const ParamVector& Trainer::params() const {
  if (!params_cache_) {
    ParamVector p{model_.layout(), std::vector<double>(model_.param_count())};
    raise_status(vnt_engine_get_params(engine_, p.values.data(), p.values.size()), "Trainer::params");
    params_cache_ = std::move(p);
  }
  return *params_cache_;
}

const World& Trainer::world() const {
  if (!world_cache_) {
    World w;
    const std::size_t in = config_.model.input_width();
    for (std::size_t i = 0; i < world_devices_.size(); ++i) {
      WorkerState ws{world_devices_[i], params(), model_.init_kernels()};
      LayerStats st;
      st.mean.assign(in, 0.0);
      st.m2.assign(in, 0.0);
      raise_status(vnt_engine_get_input_stats(engine_, (int32_t)i, &st.count, st.mean.data(), st.m2.data()),
                   "Trainer::world");
      if (st.count > 0) ws.kernels.layers["input"] = std::move(st);
      w.workers.push_back(std::move(ws));
    }
    world_cache_ = std::move(w);
  }
  return *world_cache_;
}

elastic::MigrationPlan Trainer::resize(std::vector<DeviceSpec> new_devices) {
  elastic::MigrationPlan plan = elastic::plan_resize(mapping_, std::move(new_devices));
  const World next = elastic::migrate_state(plan, world(), transport_);
  mapping_ = plan.new_mapping;
  world_devices_.clear();
  for (const auto& w : next.workers) world_devices_.push_back(w.device);
  bind_devices();
  const std::size_t in = config_.model.input_width();
  for (std::size_t i = 0; i < next.workers.size(); ++i) {
    const auto& k = next.workers[i].kernels;
    auto it = k.layers.find("input");
    std::vector<double> z(in, 0.0);
    if (it == k.layers.end() || it->second.count == 0) {
      raise_status(vnt_engine_set_input_stats(engine_, (int32_t)i, 0.0, z.data(), z.data()), "resize");
    } else {
      raise_status(vnt_engine_set_input_stats(engine_, (int32_t)i, it->second.count,
                                              it->second.mean.data(), it->second.m2.data()),
                   "resize");
    }
  }
  world_cache_.reset();
  return plan;
}

}  // namespace vnt
