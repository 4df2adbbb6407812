// vnt drop-in: Trainer (reference runner.cpp semantics) over a persistent
// B200 engine: parameters stay in HBM, the batch of each step is the same
// function of (data_seed, shuffle_seed, step) as in the reference.
//
// Processes: with a process group every process holds the same Trainer;
// device i (ascending id at construction, then new ids in order of first
// appearance) lives on process i mod P.  step() trains this process's nodes
// and reduces over the group; resize() (elastic.cpp:106-245 semantics) merges
// removed lineages into survivors and seeds added devices — on the GPU when
// both ends are here, over the engine's process pool otherwise — and changes
// which processes train (vnt_engine_set_membership), without a restart.
#include "vnt/runner.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
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
  if (world_size < 1 || rank < 0 || rank >= world_size) throw ConfigError("RunnerConfig: bad rank / world_size");
  if (world_size > 1 && !comm_ops && nccl_id.size() != 128)
    throw ConfigError("RunnerConfig: world_size > 1 needs comm_ops or a 128-byte nccl_id");
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
  o.rank = config_.rank;
  o.world_size = config_.world_size;
  o.nccl_id = config_.nccl_id.size() == 128 ? config_.nccl_id.data() : nullptr;
  o.comm_ops = config_.comm_ops;
  o.gemm_mode = config_.gemm_mode ? config_.gemm_mode : detail::engine_gemm_mode();
  o.momentum = config_.momentum;
  o.resident_rows = config_.resident_rows;
  raise_status(vnt_engine_create(&d, &o, &engine_), "Trainer");
  int32_t r = 0, n = 1;
  raise_status(vnt_engine_pool_rank(engine_, &r, &n), "Trainer");
  rank_ = r;
  procs_ = n;
  const ParamVector p = model_.init_params();
  raise_status(vnt_engine_set_params(engine_, p.values.data(), p.values.size()), "Trainer");
  place(world_devices_);
  for (std::size_t i = 0; i < local_devices().size(); ++i) {
    int32_t idx = 0;
    raise_status(vnt_engine_add_device(engine_, 1, &idx), "Trainer");
  }
  set_capacities();
  member_ = !local_devices().empty();
  if (procs_ > 1 && world_devices_.size() < (std::size_t)procs_)
    raise_status(vnt_engine_set_membership(engine_, member_ ? 1 : 0, 0), "Trainer");   // idle processes
}

Trainer::~Trainer() { vnt_engine_destroy(engine_); }

// New ids get the next process round-robin, in ascending id order.
void Trainer::place(const std::vector<DeviceSpec>& devices) {
  for (const auto& dv : devices)
    if (!placement_.count(dv.device_id)) {
      const int p = (int)(placement_.size() % (std::size_t)procs_);
      placement_.emplace(dv.device_id, p);
    }
}

std::vector<DeviceSpec> Trainer::local_devices() const {
  std::vector<DeviceSpec> mine;
  for (const auto& dv : world_devices_)
    if (placement_.at(dv.device_id) == rank_) mine.push_back(dv);
  return mine;
}

int Trainer::local_index(const std::vector<DeviceSpec>& devices, const std::string& id) const {
  int k = 0;
  for (const auto& dv : devices) {
    if (placement_.at(dv.device_id) != rank_) continue;
    if (dv.device_id == id) return k;
    ++k;
  }
  return -1;
}

void Trainer::set_capacities() {
  const auto mine = local_devices();
  for (std::size_t i = 0; i < mine.size(); ++i)
    raise_status(vnt_engine_set_device_capacity(engine_, (int32_t)i, mine[i].memory_capacity), "Trainer");
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
  StepMetrics m;
  m.step = step_;
  if (!member_) {   // this process hosts no device: the others train without it
    (void)next_batch();
    m.loss = std::numeric_limits<double>::quiet_NaN();
    ++step_;
    return m;
  }
  const Batch batch = next_batch();
  const auto mine = local_devices();
  std::map<std::string, int> index;
  for (std::size_t i = 0; i < mine.size(); ++i) index[mine[i].device_id] = (int)i;
  std::vector<int32_t> node_dev(mapping_.total_nodes(), -1);
  for (const auto& [dev, nodes] : mapping_.assignments) {
    const auto it = index.find(dev);
    if (it != index.end())
      for (auto nd : nodes) node_dev[nd] = it->second;
  }
  std::vector<std::uint64_t> sizes(mapping_.node_sizes.begin(), mapping_.node_sizes.end());
  std::vector<vnt_device_metrics> dm(std::max<std::size_t>(1, mine.size()));
  double loss = 0;
  raise_status(vnt_engine_train_step(engine_, batch.examples.data(), batch.labels.data(), batch.count,
                                     sizes.data(), node_dev.data(), (uint32_t)sizes.size(), config_.lr,
                                     &loss, dm.data()),
               "Trainer::step");
  params_cache_.reset();
  world_cache_.reset();
  m.loss = loss;
  for (std::size_t i = 0; i < mine.size(); ++i)
    m.per_device.push_back({mine[i].device_id, dm[i].waves, dm[i].examples, dm[i].peak_resident,
                            dm[i].buffer_bytes});
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
    std::vector<std::int32_t> scales(vnt_engine_scale_count(engine_));
    raise_status(vnt_engine_get_scales(engine_, scales.data(), (uint32_t)scales.size()), "Trainer::world");
    const auto mine = local_devices();
    for (std::size_t i = 0; i < mine.size(); ++i) {
      WorkerState ws{mine[i], params(), model_.init_kernels(), scales};
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

// Every process calls resize with the same list (collective).
elastic::MigrationPlan Trainer::resize(std::vector<DeviceSpec> new_devices) {
  elastic::MigrationPlan plan = elastic::plan_resize(mapping_, std::move(new_devices));
  const std::vector<DeviceSpec> before = world_devices_;
  const std::vector<DeviceSpec> after = sorted_devices(plan.new_mapping.devices);
  if (plan.merge_sources.empty() && plan.state_sources.empty() && plan.moves.empty() &&
      before.size() == after.size()) {
    mapping_ = plan.new_mapping;
    world_devices_ = after;
    set_capacities();
    return plan;
  }
  place(after);
  const bool was_member = member_;
  // 1. removed lineages into their survivors, in the plan's order: on the GPU
  //    when both live here, over the process pool otherwise
  for (const auto& [survivor, removed] : plan.merge_sources)
    for (const auto& gone : removed) {
      const int from = placement_.at(gone), to = placement_.at(survivor);
      if (from == rank_ && to == rank_) {
        const int32_t n = (int32_t)vnt_engine_device_count(engine_);
        std::vector<int32_t> same(n);
        for (int32_t k = 0; k < n; ++k) same[k] = k;
        const int32_t pair[2] = {local_index(before, gone), local_index(before, survivor)};
        raise_status(vnt_engine_remap_devices(engine_, (uint32_t)n, same.data(), 1, pair), "Trainer::resize");
      } else if (from == rank_) {
        raise_status(vnt_engine_send_lineage(engine_, local_index(before, gone), to), "Trainer::resize");
      } else if (to == rank_) {
        raise_status(vnt_engine_recv_lineage(engine_, from, local_index(before, survivor), 1), "Trainer::resize");
      }
    }
  // 2. this process's new device list: survivors keep their lineage, added
  //    devices seeded here start as a copy of their (post-merge) survivor
  std::vector<int32_t> src;
  for (const auto& dv : after) {
    if (placement_.at(dv.device_id) != rank_) continue;
    int32_t s0 = local_index(before, dv.device_id);   // a survivor hosted here
    if (s0 < 0) {
      const auto it = plan.state_sources.find(dv.device_id);
      if (it != plan.state_sources.end() && placement_.at(it->second) == rank_) s0 = local_index(before, it->second);
    }
    src.push_back(s0);
  }
  raise_status(vnt_engine_remap_devices(engine_, (uint32_t)src.size(), src.data(), 0, nullptr), "Trainer::resize");
  world_devices_ = after;
  mapping_ = plan.new_mapping;
  // 3. which processes train now: the replica state comes from the lowest
  //    process that trained before
  member_ = !local_devices().empty();
  if (procs_ > 1) {
    int source = procs_;
    for (const auto& dv : before) source = std::min(source, placement_.at(dv.device_id));
    (void)was_member;
    raise_status(vnt_engine_set_membership(engine_, member_ ? 1 : 0, source), "Trainer::resize");
  }
  // 4. added devices seeded from a survivor on another process
  for (const auto& [added, survivor] : plan.state_sources) {
    const int from = placement_.at(survivor), to = placement_.at(added);
    if (from == to) continue;
    if (from == rank_)
      raise_status(vnt_engine_send_lineage(engine_, local_index(after, survivor), to), "Trainer::resize");
    else if (to == rank_)
      raise_status(vnt_engine_recv_lineage(engine_, from, local_index(after, added), 0), "Trainer::resize");
  }
  set_capacities();
  params_cache_.reset();
  world_cache_.reset();
  return plan;
}

}  // namespace vnt
