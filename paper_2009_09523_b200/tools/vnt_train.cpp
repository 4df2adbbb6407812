// `vnt train` on the B200 engine: the reference CLI's train command
// (tools/vnt.cpp:52-152, docs/schemas/train.schema.json) over the drop-in
// vnt::Trainer.  Same config keys (unknown keys rejected), same outputs
// (StepMetrics JSONL, params JSON {"layout","values"}), same --compare-against
// semantics and exit codes (0 ok, 2 config/shape, 3 capacity, 4 divergence, 1
// other).  Extension keys: "gemm_mode" (auto|ffma|tf32|3xf16; 3xtf32 = 3xf16), "momentum".
// The reference's `profile` / `solve` commands drive the cluster planner,
// which is out of scope here.
//
//   vnt_train train --config cfg.json [--json] [--seed N] [--compare-against params.json]
#include <cmath>
#include <fstream>
#include <iostream>
#include <optional>
#include <set>
#include <sstream>
#include <string>

#include <filesystem>

#include "nlohmann/json.hpp"
#include "vnt/errors.hpp"
#include "vnt/runner.hpp"
#include "vnt_engine.h"

using json = nlohmann::json;

namespace {

constexpr int kExitConfig = 2, kExitCapacity = 3, kExitDivergence = 4;

struct Divergence : vnt::Error {
  using Error::Error;
};

// Strict object access: every key must be consumed or it is an error.
class Keys {
 public:
  Keys(const json& j, std::string what) : j_(j), what_(std::move(what)) {
    if (!j.is_object()) throw vnt::ConfigError(what_ + ": expected an object");
  }
  const json& need(const std::string& k) {
    if (!j_.contains(k)) throw vnt::ConfigError(what_ + ": missing key '" + k + "'");
    used_.insert(k);
    return j_.at(k);
  }
  const json* maybe(const std::string& k) {
    if (!j_.contains(k)) return nullptr;
    used_.insert(k);
    return &j_.at(k);
  }
  void finish() const {
    for (auto it = j_.begin(); it != j_.end(); ++it)
      if (!used_.count(it.key())) throw vnt::ConfigError(what_ + ": unknown key '" + it.key() + "'");
  }

 private:
  const json& j_;
  std::string what_;
  std::set<std::string> used_;
};

vnt::DeviceSpec device_of(const json& j) {
  Keys k(j, "device");
  vnt::DeviceSpec d{k.need("device_id").get<std::string>(), k.need("device_type").get<std::string>(),
                    k.need("memory_capacity").get<std::size_t>()};
  k.finish();
  if (d.device_id.empty()) throw vnt::ConfigError("device: empty device_id");
  if (d.memory_capacity == 0) throw vnt::ConfigError("device " + d.device_id + ": zero memory_capacity");
  return d;
}

std::vector<vnt::DeviceSpec> devices_of(const json& j) {
  if (!j.is_array() || j.empty()) throw vnt::ConfigError("devices: expected a non-empty array");
  std::vector<vnt::DeviceSpec> v;
  for (const auto& d : j) v.push_back(device_of(d));
  return v;
}

json params_json(const vnt::ParamVector& p) {
  json layout = json::array();
  for (const auto& e : p.layout->entries) layout.push_back(json{{"name", e.name}, {"shape", e.shape}});
  return json{{"layout", layout}, {"values", p.values}};
}

std::vector<double> params_values(const json& j, std::size_t expect) {
  Keys k(j, "params");
  (void)k.need("layout");
  auto v = k.need("values").get<std::vector<double>>();
  k.finish();
  if (v.size() != expect) throw vnt::ShapeError("--compare-against: parameter layouts differ");
  return v;
}

json load(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw vnt::ConfigError("cannot open " + path);
  try {
    return json::parse(f);
  } catch (const json::exception& e) {
    throw vnt::ConfigError(path + ": " + e.what());
  }
}

void write(const std::string& path, const std::string& text) {
  const auto parent = std::filesystem::path(path).parent_path();
  if (!parent.empty()) std::filesystem::create_directories(parent);
  std::ofstream f(path);
  if (!f) throw vnt::ConfigError("cannot write " + path);
  f << text;
}

int gemm_mode_of(const std::string& s) {
  if (s == "auto") return VNT_GEMM_AUTO;
  if (s == "ffma") return VNT_GEMM_FFMA;
  if (s == "tf32") return VNT_GEMM_TF32;
  if (s == "3xf16" || s == "3xtf32") return VNT_GEMM_3XF16;
  throw vnt::ConfigError("unknown gemm_mode: " + s);
}

int cmd_train(const std::string& cfg_path, bool json_out, std::optional<std::uint64_t> seed,
              const std::string& compare) {
  const json cfg = load(cfg_path);
  Keys k(cfg, "train config");
  vnt::RunnerConfig rc;
  {
    Keys w(k.need("workload"), "workload");
    rc.model.layer_widths = w.need("layer_widths").get<std::vector<std::size_t>>();
    rc.model.activation = vnt::activation_from_string(w.need("activation").get<std::string>());
    rc.model.loss = vnt::loss_from_string(w.need("loss").get<std::string>());
    rc.model.seed = w.need("seed").get<std::uint64_t>();
    w.finish();
  }
  rc.global_batch = k.need("global_batch").get<std::size_t>();
  rc.virtual_nodes = k.need("virtual_nodes").get<std::size_t>();
  const auto steps = k.need("steps").get<std::size_t>();
  rc.lr = k.need("lr").get<double>();
  rc.devices = devices_of(k.need("devices"));
  if (auto* v = k.maybe("data_seed")) rc.data_seed = v->get<std::uint64_t>();
  if (auto* v = k.maybe("dataset_size")) rc.dataset_size = v->get<std::size_t>();
  if (auto* v = k.maybe("shuffle_epochs")) rc.shuffle_epochs = v->get<bool>();
  if (auto* v = k.maybe("shuffle_seed")) rc.shuffle_seed = v->get<std::uint64_t>();
  if (auto* v = k.maybe("parallel_devices")) rc.parallel_devices = v->get<bool>();
  if (auto* v = k.maybe("prefetch")) rc.prefetch = v->get<bool>();
  if (auto* v = k.maybe("gemm_mode")) rc.gemm_mode = gemm_mode_of(v->get<std::string>());
  if (auto* v = k.maybe("momentum")) rc.momentum = v->get<double>();
  std::vector<vnt::elastic::ResizePoint> schedule;
  if (auto* v = k.maybe("resize_schedule")) {
    for (const auto& pt : *v) {
      Keys r(pt, "resize point");
      schedule.push_back({r.need("step").get<std::uint64_t>(), devices_of(r.need("devices"))});
      r.finish();
    }
  }
  double tolerance = 0.0;
  if (auto* v = k.maybe("compare_tolerance")) tolerance = v->get<double>();
  std::string metrics_out, params_out;
  if (auto* v = k.maybe("metrics_out")) metrics_out = v->get<std::string>();
  if (auto* v = k.maybe("params_out")) params_out = v->get<std::string>();
  k.finish();
  if (seed) rc.model.seed = rc.data_seed = *seed;

  vnt::Trainer trainer(rc);
  std::string lines;
  std::size_t cur = 0;
  double last = 0.0;
  for (std::uint64_t s = 0; s < steps; ++s) {
    while (cur < schedule.size() && schedule[cur].step == s) trainer.resize(schedule[cur++].devices);
    const vnt::StepMetrics m = trainer.step();
    last = m.loss;
    json pd = json::array();
    for (const auto& d : m.per_device)
      pd.push_back(json{{"device_id", d.device_id}, {"waves", d.waves}, {"examples", d.examples},
                        {"peak_resident", d.peak_resident}, {"buffer_bytes", d.buffer_bytes}});
    lines += json{{"step", m.step}, {"loss", m.loss}, {"per_device", pd}}.dump() + "\n";
  }
  if (!metrics_out.empty()) write(metrics_out, lines);
  if (!params_out.empty()) write(params_out, params_json(trainer.params()).dump(2) + "\n");

  json summary{{"steps", steps}, {"final_loss", last}, {"devices", trainer.world().workers.size()}};
  if (!compare.empty()) {
    const auto other = params_values(load(compare), trainer.params().values.size());
    double mx = 0.0;
    bool bitwise = true;
    const auto& mine = trainer.params().values;
    for (std::size_t i = 0; i < other.size(); ++i) {
      mx = std::max(mx, std::abs(mine[i] - other[i]));
      bitwise &= std::memcmp(&mine[i], &other[i], sizeof(double)) == 0;
    }
    summary["max_divergence"] = mx;
    summary["bitwise_identical"] = bitwise;
    if (mx > tolerance) {
      if (json_out) std::cout << summary.dump() << "\n";
      throw Divergence("parameter divergence " + json(mx).dump() + " exceeds tolerance " +
                       json(tolerance).dump());
    }
  }
  if (json_out) {
    std::cout << summary.dump() << "\n";
  } else {
    std::cout << "trained " << steps << " steps on " << trainer.world().workers.size()
              << " devices, final loss " << json(last).dump() << "\n";
  }
  return 0;
}

vnt::ModelSpec model_of(const json& j) {
  Keys w(j, "workload");
  vnt::ModelSpec m;
  m.layer_widths = w.need("layer_widths").get<std::vector<std::size_t>>();
  m.activation = vnt::activation_from_string(w.need("activation").get<std::string>());
  m.loss = vnt::loss_from_string(w.need("loss").get<std::string>());
  m.seed = w.need("seed").get<std::uint64_t>();
  w.finish();
  return m;
}

}  // namespace

int main(int argc, char** argv) {
  std::string cmd, cfg, compare;
  bool json_out = false;
  std::optional<std::uint64_t> seed;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw vnt::ConfigError(a + " needs a value");
      return argv[++i];
    };
    try {
      if (a == "--config") cfg = next();
      else if (a == "--json") json_out = true;
      else if (a == "--seed") seed = std::stoull(next());
      else if (a == "--compare-against") compare = next();
      else if (cmd.empty() && a[0] != '-') cmd = a;
      else throw vnt::ConfigError("unknown argument " + a);
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return kExitConfig;
    }
  }
  if (cmd != "train" || cfg.empty()) {
    std::cerr << "usage: vnt_train train --config FILE [--json] [--seed N] [--compare-against FILE]\n";
    return kExitConfig;
  }
  try {
    return cmd_train(cfg, json_out, seed, compare);
  } catch (const Divergence& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitDivergence;
  } catch (const vnt::CapacityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitCapacity;
  } catch (const vnt::ConfigError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitConfig;
  } catch (const vnt::ShapeError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitConfig;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
