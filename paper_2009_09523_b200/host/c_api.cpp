// C-ABI over the C++ drop-in (include/vnt_trainer.h).
#include <cstring>
#include <memory>
#include <string>

#include "vnt/errors.hpp"
#include "vnt/hetero.hpp"
#include "vnt/runner.hpp"
#include "vnt_trainer.h"

struct vnt_trainer {
  std::unique_ptr<vnt::Trainer> t;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    return f();
  } catch (const vnt::CapacityError& e) {
    g_err = e.what();
    return VNT_ERR_CAPACITY;
  } catch (const vnt::ConfigError& e) {
    g_err = e.what();
    return VNT_ERR_CONFIG;
  } catch (const vnt::ShapeError& e) {
    g_err = e.what();
    return VNT_ERR_SHAPE;
  } catch (const vnt::ConsistencyError& e) {
    g_err = e.what();
    return VNT_ERR_CONSISTENCY;
  } catch (const vnt::MigrationError& e) {
    g_err = e.what();
    return VNT_ERR_MIGRATION;
  } catch (const vnt::InfeasibleError& e) {
    g_err = e.what();
    return VNT_ERR_INFEASIBLE;
  } catch (const vnt::ProfileError& e) {
    g_err = e.what();
    return VNT_ERR_PROFILE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VNT_ERR_INTERNAL;
  }
}

std::vector<vnt::DeviceSpec> specs(const vnt_device_spec* d, uint32_t n) {
  std::vector<vnt::DeviceSpec> v;
  for (uint32_t i = 0; i < n; ++i)
    v.push_back({d[i].device_id ? d[i].device_id : "", d[i].device_type ? d[i].device_type : "",
                 d[i].memory_capacity});
  return v;
}
}  // namespace

extern "C" {

const char* vnt_host_last_error(void) { return g_err.c_str(); }

int vnt_trainer_create(const vnt_runner_config* c, vnt_trainer** out) {
  return guard([&] {
    vnt::RunnerConfig rc;
    rc.model.layer_widths.assign(c->layer_widths, c->layer_widths + c->num_widths);
    rc.model.activation = static_cast<vnt::Activation>(c->activation);
    rc.model.loss = static_cast<vnt::Loss>(c->loss);
    rc.model.seed = c->seed;
    rc.global_batch = c->global_batch;
    rc.virtual_nodes = c->virtual_nodes;
    rc.lr = c->lr;
    rc.data_seed = c->data_seed;
    rc.dataset_size = c->dataset_size;
    rc.shuffle_epochs = c->shuffle_epochs != 0;
    rc.shuffle_seed = c->shuffle_seed;
    rc.devices = specs(c->devices, c->num_devices);
    rc.parallel_devices = c->parallel_devices != 0;
    rc.prefetch = c->prefetch != 0;
    rc.gemm_mode = c->gemm_mode;
    rc.momentum = c->momentum;
    rc.comm_ops = c->comm_ops;
    if (c->nccl_id) rc.nccl_id.assign(c->nccl_id, c->nccl_id + 128);
    rc.rank = c->rank;
    rc.world_size = c->world_size < 1 ? 1 : c->world_size;
    rc.cuda_device = c->cuda_device;
    rc.resident_rows = c->resident_rows;
    auto t = std::make_unique<vnt_trainer>();
    t->t = std::make_unique<vnt::Trainer>(rc);
    *out = t.release();
    return VNT_OK;
  });
}

void vnt_trainer_destroy(vnt_trainer* t) { delete t; }

uint64_t vnt_trainer_param_count(const vnt_trainer* t) { return t->t->model().param_count(); }

int vnt_trainer_step(vnt_trainer* t, double* loss, vnt_device_metrics* pd, uint32_t cap) {
  return guard([&] {
    const auto m = t->t->step();
    if (loss) *loss = m.loss;
    for (uint32_t i = 0; pd && i < cap && i < m.per_device.size(); ++i)
      pd[i] = {m.per_device[i].waves, m.per_device[i].examples, m.per_device[i].peak_resident,
               m.per_device[i].buffer_bytes};
    return VNT_OK;
  });
}

int vnt_trainer_params(vnt_trainer* t, double* out, uint64_t n) {
  return guard([&] {
    const auto& p = t->t->params();
    if (n != p.values.size()) throw vnt::ShapeError("params size mismatch");
    std::memcpy(out, p.values.data(), n * sizeof(double));
    return VNT_OK;
  });
}

int vnt_trainer_resize(vnt_trainer* t, const vnt_device_spec* d, uint32_t n) {
  return guard([&] {
    t->t->resize(specs(d, n));
    return VNT_OK;
  });
}

uint32_t vnt_trainer_device_count(const vnt_trainer* t) {
  return (uint32_t)t->t->world().workers.size();
}

int vnt_trainer_input_stats(vnt_trainer* t, uint32_t idx, double* count, double* mean, double* m2) {
  return guard([&] {
    const auto& w = t->t->world().workers.at(idx);
    const std::size_t in = t->t->model().spec().input_width();
    auto it = w.kernels.layers.find("input");
    if (it == w.kernels.layers.end()) {
      *count = 0;
      std::memset(mean, 0, in * sizeof(double));
      std::memset(m2, 0, in * sizeof(double));
      return VNT_OK;
    }
    *count = it->second.count;
    std::memcpy(mean, it->second.mean.data(), in * sizeof(double));
    std::memcpy(m2, it->second.m2.data(), in * sizeof(double));
    return VNT_OK;
  });
}

int vnt_synth_batch(uint64_t seed, uint64_t n, uint64_t in, uint64_t out, uint64_t start,
                    uint64_t count, double* x, double* y) {
  return guard([&] {
    const vnt::Batch b = vnt::SynthDataset(seed, n, in, out).sequential_batch(start, count);
    std::memcpy(x, b.examples.data(), b.examples.size() * sizeof(double));
    std::memcpy(y, b.labels.data(), b.labels.size() * sizeof(double));
    return VNT_OK;
  });
}

int vnt_init_params(const uint64_t* widths, uint32_t nw, uint64_t seed, double* out) {
  return guard([&] {
    vnt::ModelSpec s;
    s.layer_widths.assign(widths, widths + nw);
    s.seed = seed;
    const auto p = vnt::Model(s).init_params();
    std::memcpy(out, p.values.data(), p.values.size() * sizeof(double));
    return VNT_OK;
  });
}


int vnt_hetero_profile_device(const uint64_t* widths, uint32_t nw, int32_t activation,
                              int32_t loss, uint64_t seed, const char* device_type,
                              uint64_t memory_capacity, const uint64_t* batch_sizes, uint32_t nb,
                              uint64_t steps, uint64_t warmup_cutoff, int32_t cuda_device,
                              int32_t gemm_mode, uint64_t* out_batch, double* out_time,
                              uint32_t* out_npts, double* out_comm) {
  return guard([&] {
    vnt::ModelSpec spec;
    spec.layer_widths.assign(widths, widths + nw);
    spec.activation = static_cast<vnt::Activation>(activation);
    spec.loss = static_cast<vnt::Loss>(loss);
    spec.seed = seed;
    vnt::hetero::ProfileOptions o;
    o.steps = steps;
    o.warmup_cutoff = warmup_cutoff;
    const auto r = vnt::hetero::profile_device(
        spec, device_type, memory_capacity, std::vector<std::size_t>(batch_sizes, batch_sizes + nb), o,
        cuda_device, gemm_mode);
    *out_npts = (uint32_t)r.curve.points.size();
    for (std::size_t k = 0; k < r.curve.points.size(); ++k) {
      out_batch[k] = r.curve.points[k].batch_size;
      out_time[k] = r.curve.points[k].step_time_s;
    }
    *out_comm = r.curve.comm_overhead_s;
    return VNT_OK;
  });
}

}  // extern "C"
