// Internal: the engine bound to a vnt::Model for the compatibility free
// functions (Model::forward_backward, device_step, train_step).
#pragma once

#include <mutex>

#include "vnt/model.hpp"
#include "vnt_engine.h"

namespace vnt::detail {

struct GpuModel {
  explicit GpuModel(const ModelSpec& spec);
  ~GpuModel();
  GpuModel(const GpuModel&) = delete;
  GpuModel& operator=(const GpuModel&) = delete;

  // Makes at least n logical devices exist with the given capacities.
  void ensure_devices(const std::vector<std::size_t>& capacities);
  // Skipped when the engine already holds exactly these values (the last
  // upload or download): the reference API passes params by value on every
  // call, the engine keeps them resident.
  void upload_params(const std::vector<double>& values);
  std::vector<double> download_params();
  void set_stats(int dev, const StatefulKernelState& k);
  void get_stats(int dev, StatefulKernelState& k);

  std::mutex mu;
  vnt_engine* eng = nullptr;
  std::vector<double> resident;   // host copy of the engine's parameters (if known)
  bool resident_valid = false;
  std::size_t in_width = 0;
  int ndev = 0;
};

int engine_gemm_mode();  // VNT_GEMM_MODE env: auto|ffma|tf32|3xf16 (3xtf32: old name)

}  // namespace vnt::detail
