// Host-side drop-in behaviour (no GPU): RNG/data determinism, layout,
// mapping and elastic planning, exact sums, kernel statistics.  Cases follow
// the reference suites (test_rng.cpp, test_data.cpp, test_virtual_exec.cpp:32-55,
// test_elastic.cpp:42-150, test_model.cpp:54-66,212-267).
#include <algorithm>
#include <numeric>

#include "check.hpp"
#include "vnt/elastic.hpp"
#include "vnt/errors.hpp"
#include "vnt/rng.hpp"
#include "vnt/runner.hpp"

using namespace vnt;

static std::vector<DeviceSpec> gpus(std::size_t n, std::size_t cap = 1024) {
  std::vector<DeviceSpec> d;
  for (std::size_t i = 0; i < n; ++i) d.push_back({"gpu" + std::to_string(i), "B200", cap});
  return d;
}

TEST_CASE("rng is a pure function of key and counter") {
  const CounterRng a(7), b(7);
  CHECK(a.bits(12345) == b.bits(12345));
  CHECK(a.split("x").bits(3) == b.split("x").bits(3));
  CHECK(a.split("x").bits(3) != a.split("y").bits(3));
  for (std::uint64_t c = 0; c < 1000; ++c) {
    const double u = a.uniform(c);
    CHECK(u >= 0.0 && u < 1.0);
    CHECK(std::isfinite(a.normal(c)));
  }
  CHECK_THROWS_AS(a.below(1, 0), ConfigError);
  auto p = random_permutation(a, 50);
  std::sort(p.begin(), p.end());
  for (std::uint64_t i = 0; i < 50; ++i) CHECK(p[i] == i);
}

TEST_CASE("synthetic labels are distributions and order independent") {
  SynthDataset d(3, 40, 5, 4);
  const Batch b = d.sequential_batch(38, 5);  // wraps
  CHECK(b.ids[2] == 0);
  for (std::size_t r = 0; r < b.count; ++r) {
    double s = 0;
    for (double v : b.label(r)) s += v;
    CHECK(std::abs(s - 1.0) < 1e-12);
  }
  std::vector<std::uint64_t> ids = {7, 3};
  const Batch c = d.batch(ids);
  const Batch e = d.sequential_batch(3, 1);
  CHECK(std::equal(c.example(1).begin(), c.example(1).end(), e.example(0).begin()));
  CHECK_THROWS_AS(d.batch(std::vector<std::uint64_t>{40}), ConfigError);
  CHECK_THROWS_AS(SynthDataset(1, 0, 2, 2), ConfigError);
}

TEST_CASE("layout and init follow the reference layout") {
  ModelSpec s{{4, 16, 4}, Activation::kTanh, Loss::kMse, 11};
  Model m(s);
  CHECK(m.param_count() == 4 * 16 + 16 + 16 * 4 + 4);
  CHECK(m.layout()->entries[1].name == "layer0/bias");
  CHECK(m.layout()->entries[2].offset == 80);
  const auto p = m.init_params();
  CHECK(p.values[64] == 0.0 && p.values[79] == 0.0);  // biases start at zero
  CHECK(p.bitwise_equal(m.init_params()));
  CHECK_THROWS_AS(Model(ModelSpec{{4}, Activation::kTanh, Loss::kMse, 0}), ConfigError);
  CHECK_THROWS_AS(activation_from_string("gelu"), ConfigError);
}

TEST_CASE("uniform mapping shapes and capacity errors name the device") {
  const auto m = make_uniform_mapping(16, 16, gpus(4));
  for (const auto& [d, nodes] : m.assignments) CHECK(nodes.size() == 4);
  const auto big = make_uniform_mapping(8192, 32, gpus(1, 256));
  CHECK(big.assignments.at("gpu0").size() == 32);
  CHECK_THROWS_WITH_AS(make_uniform_mapping(64, 4, gpus(2, 8)), "gpu0", CapacityError);
  CHECK_THROWS_AS(make_uniform_mapping(10, 3, gpus(1)), ConfigError);
  CHECK_THROWS_AS(make_uniform_mapping(8, 2, gpus(4)), ConfigError);
}

TEST_CASE("resize planning re-deals nodes and names state sources") {
  const auto m = make_uniform_mapping(16, 8, gpus(2));
  const auto plan = elastic::plan_resize(m, gpus(4));
  for (const auto& [d, nodes] : plan.new_mapping.assignments) CHECK(nodes.size() == 2);
  CHECK(plan.state_sources.size() == 2);
  CHECK(plan.state_sources.at("gpu2") == "gpu0");
  CHECK(plan.state_sources.at("gpu3") == "gpu1");
  const auto same = elastic::plan_resize(m, gpus(2));
  CHECK(same.moves.empty() && same.state_sources.empty() && same.merge_sources.empty());
  const auto shrink = elastic::plan_resize(make_uniform_mapping(16, 16, gpus(16)), gpus(4));
  for (const auto& [d, nodes] : shrink.new_mapping.assignments) CHECK(nodes.size() == 4);
  auto small = make_uniform_mapping(16, 4, gpus(4, 8));
  CHECK_THROWS_WITH_AS(elastic::plan_resize(small, gpus(1, 2)), "virtual node", CapacityError);
  elastic::ResizeRequest req{"job", {}, 5};
  CHECK_THROWS_AS(req.validate(4), ConfigError);
}

TEST_CASE("exact accumulators are order independent") {
  ExactAccumulator a, b;
  const double v[] = {1e100, 1.0, -1e100, 1e-300, 3.0, -2.5e-17};
  for (double x : v) a.add(x);
  for (int i = 5; i >= 0; --i) b.add(v[i]);
  CHECK(a.total() == b.total());
  CHECK(a.total() == 4.0);
  ExactAccumulator c;
  c.add(0.1);
  c.add(0.2);
  CHECK(c.total() == 0.30000000000000004);
}

TEST_CASE("kernel statistics combine exactly like a from-scratch pass") {
  std::vector<double> rows = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10};
  LayerStats whole, parts;
  whole.observe(5, 2, rows);
  parts.observe(2, 2, std::span<const double>(rows).subspan(0, 4));
  parts.observe(3, 2, std::span<const double>(rows).subspan(4, 6));
  CHECK(whole.count == parts.count);
  for (int j = 0; j < 2; ++j) {
    CHECK(std::abs(whole.mean[j] - parts.mean[j]) < 1e-12);
    CHECK(std::abs(whole.variance()[j] - parts.variance()[j]) < 1e-12);
  }
}

TEST_CASE("runner config validation") {
  RunnerConfig c;
  c.model = ModelSpec{{3, 6, 2}, Activation::kTanh, Loss::kMse, 1};
  c.global_batch = 10;
  c.virtual_nodes = 3;
  c.devices = gpus(1);
  CHECK_THROWS_AS(c.validate(), ConfigError);
  c.virtual_nodes = 2;
  c.lr = 0;
  CHECK_THROWS_AS(c.validate(), ConfigError);
  c.lr = 0.1;
  c.shuffle_epochs = true;
  c.dataset_size = 15;
  CHECK_THROWS_AS(c.validate(), ConfigError);
}

TEST_MAIN()
