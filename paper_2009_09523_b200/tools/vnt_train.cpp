// `vnt train | profile | solve` on the B200 engine: the reference CLI's
// commands (tools/vnt.cpp:52-263, docs/schemas/{train,profile,solve}.schema.json)
// over the drop-in vnt::Trainer and vnt::hetero.  Same config keys (unknown keys
// rejected), same outputs (StepMetrics JSONL, params JSON {"layout","values"},
// profile curves, assignment JSON), same --compare-against semantics and exit
// codes (0 ok, 2 config/shape, 3 capacity, 4 divergence, 5 infeasible, 1
// other).  Extension keys: train "gemm_mode" (auto|ffma|tf32|3xtf32),
// "momentum"; profile device model "measure": true (time the workload on this
// B200 with hetero::profile_device instead of the synthetic cost model).
//
//   vnt_train train --config cfg.json [--json] [--seed N] [--compare-against params.json]
//   vnt_train profile --config cfg.json [--json]
//   vnt_train solve --config cfg.json [--json] [--explain]
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
#include "vnt/hetero.hpp"
#include "vnt/runner.hpp"
#include "vnt_engine.h"

using json = nlohmann::json;

namespace {

constexpr int kExitConfig = 2, kExitCapacity = 3, kExitDivergence = 4, kExitInfeasible = 5;

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
  if (s == "3xtf32") return VNT_GEMM_3XTF32;
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

json curve_json(const vnt::hetero::ProfileCurve& c) {
  json pts = json::array();
  for (const auto& p : c.points) pts.push_back(json{{"batch_size", p.batch_size}, {"step_time_s", p.step_time_s}});
  return json{{"device_type", c.device_type}, {"comm_overhead_s", c.comm_overhead_s}, {"points", pts}};
}

vnt::hetero::ProfileCurve curve_of(const json& j) {
  Keys k(j, "profile");
  vnt::hetero::ProfileCurve c;
  c.device_type = k.need("device_type").get<std::string>();
  c.comm_overhead_s = k.need("comm_overhead_s").get<double>();
  for (const json& pj : k.need("points")) {
    Keys pk(pj, "profile point");
    vnt::hetero::ProfilePoint p{pk.need("batch_size").get<std::size_t>(), pk.need("step_time_s").get<double>()};
    pk.finish();
    if (p.batch_size == 0 || !(p.step_time_s > 0))
      throw vnt::ConfigError("profile point: batch size and step time must be positive");
    c.points.push_back(p);
  }
  k.finish();
  return c;
}

json assignment_json(const vnt::hetero::HeteroAssignment& a) {
  json types = json::array();
  for (const auto& t : a.types)
    types.push_back(json{{"device_type", t.device_type}, {"count", t.devices_used},
                         {"per_device_batch", t.per_device_batch}, {"virtual_nodes", t.virtual_nodes}});
  return json{{"global_batch", a.global_batch}, {"predicted_step_time_s", a.predicted_step_time_s},
              {"types", types}};
}

// `vnt profile` (tools/vnt.cpp:154-197): one curve per device model over the
// candidate grid up to max_batch, written to <out_dir>/<device_type>.json.
int cmd_profile(const std::string& cfg_path, bool json_out) {
  const json cfg = load(cfg_path);
  Keys k(cfg, "profile config");
  const vnt::ModelSpec workload = model_of(k.need("workload"));
  const auto max_batch = k.need("max_batch").get<std::size_t>();
  struct Model {
    vnt::hetero::DeviceCostModel cost;
    bool measure = false;
  };
  std::vector<Model> models;
  for (const json& mj : k.need("device_models")) {
    Keys m(mj, "device model");
    Model md;
    md.cost.device_type = m.need("device_type").get<std::string>();
    md.cost.fixed_overhead_s = m.need("fixed_overhead_s").get<double>();
    md.cost.per_example_cost_s = m.need("per_example_cost_s").get<double>();
    md.cost.comm_s = m.need("comm_s").get<double>();
    md.cost.memory_capacity = m.need("memory_capacity").get<std::size_t>();
    if (auto* v = m.maybe("first_step_multiplier")) md.cost.first_step_multiplier = v->get<double>();
    if (auto* v = m.maybe("measure")) md.measure = v->get<bool>();
    m.finish();
    md.cost.validate();
    models.push_back(md);
  }
  vnt::hetero::ProfileOptions opt;
  if (auto* v = k.maybe("steps")) opt.steps = v->get<std::size_t>();
  if (auto* v = k.maybe("data_seed")) opt.data_seed = v->get<std::uint64_t>();
  const auto out_dir = k.need("out_dir").get<std::string>();
  k.finish();
  if (models.empty()) throw vnt::ConfigError("profile: no device models");
  std::filesystem::create_directories(out_dir);
  const auto grid = vnt::hetero::candidate_batch_sizes(max_batch);
  json written = json::array();
  for (const auto& md : models) {
    const auto r = md.measure ? vnt::hetero::profile_device(workload, md.cost.device_type,
                                                            md.cost.memory_capacity, grid, opt)
                              : vnt::hetero::profile(workload, md.cost, grid, opt);
    for (const auto& w : r.warnings) std::cerr << "warning: " << w << "\n";
    if (r.curve.points.empty())
      throw vnt::ConfigError("profile: no batch size fits device type " + md.cost.device_type +
                             "; curve would be empty");
    const std::string path = out_dir + "/" + md.cost.device_type + ".json";
    write(path, curve_json(r.curve).dump(2) + "\n");
    written.push_back(path);
  }
  if (json_out) {
    std::cout << json{{"profiles", written}}.dump() << "\n";
  } else {
    for (const auto& p : written) std::cout << "wrote " << p.get<std::string>() << "\n";
  }
  return 0;
}

// `vnt solve` (tools/vnt.cpp:199-263): heterogeneous assignment from curves.
int cmd_solve(const std::string& cfg_path, bool json_out, bool explain) {
  const json cfg = load(cfg_path);
  Keys k(cfg, "solve config");
  std::vector<vnt::hetero::ProfileCurve> curves;
  for (const json& p : k.need("profiles")) curves.push_back(curve_of(load(p.get<std::string>())));
  vnt::hetero::DevicePool pool;
  const json& pj = k.need("pool");
  if (!pj.is_object()) throw vnt::ConfigError("solve: pool must be an object");
  for (auto it = pj.begin(); it != pj.end(); ++it) {
    Keys e(it.value(), "pool entry " + it.key());
    pool.entries[it.key()] = {e.need("count").get<std::size_t>(), e.need("memory_capacity").get<std::size_t>()};
    e.finish();
  }
  const auto global_batch = k.need("global_batch").get<std::size_t>();
  vnt::hetero::SolveOptions opt;
  opt.collect_candidates = explain;
  if (auto* v = k.maybe("max_virtual_nodes")) opt.max_virtual_nodes = v->get<std::size_t>();
  std::string out;
  if (auto* v = k.maybe("out")) out = v->get<std::string>();
  k.finish();
  const auto r = vnt::hetero::solve(curves, pool, global_batch, opt);
  const json a = assignment_json(r.best);
  if (!out.empty()) write(out, a.dump(2) + "\n");
  if (json_out) {
    json payload{{"assignment", a}};
    if (explain) {
      json table = json::array();
      for (const auto& c : r.candidates) table.push_back(assignment_json(c));
      payload["candidates"] = table;
    }
    std::cout << payload.dump() << "\n";
  } else {
    std::cout << "predicted step time: " << json(r.best.predicted_step_time_s).dump() << " s\n";
    for (const auto& t : r.best.types)
      std::cout << "  " << t.device_type << ": n=" << t.devices_used << " b=" << t.per_device_batch
                << " v=" << t.virtual_nodes << "\n";
    if (explain) std::cout << "evaluated " << r.candidates.size() << " candidates\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::string cmd, cfg, compare;
  bool json_out = false, explain = false;
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
      else if (a == "--explain") explain = true;
      else if (a == "--seed") seed = std::stoull(next());
      else if (a == "--compare-against") compare = next();
      else if (cmd.empty() && a[0] != '-') cmd = a;
      else throw vnt::ConfigError("unknown argument " + a);
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return kExitConfig;
    }
  }
  if ((cmd != "train" && cmd != "profile" && cmd != "solve") || cfg.empty()) {
    std::cerr << "usage: vnt_train train --config FILE [--json] [--seed N] [--compare-against FILE]\n"
                 "       vnt_train profile --config FILE [--json]\n"
                 "       vnt_train solve --config FILE [--json] [--explain]\n";
    return kExitConfig;
  }
  try {
    if (cmd == "profile") return cmd_profile(cfg, json_out);
    if (cmd == "solve") return cmd_solve(cfg, json_out, explain);
    return cmd_train(cfg, json_out, seed, compare);
  } catch (const Divergence& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitDivergence;
  } catch (const vnt::CapacityError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitCapacity;
  } catch (const vnt::InfeasibleError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitInfeasible;
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
