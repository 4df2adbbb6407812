// The C++ drop-in API on the GPU: the reference's own test cases
// (test_virtual_exec.cpp, test_elastic.cpp) run against vnt:: backed by the
// B200 engine.  Exactness claims that hold bit-for-bit in the reference hold
// bit-for-bit here (mapping invariance, serial == parallel, resize
// transparency); fp64-oracle comparisons use the engine's fp32 tolerance.
#include <cmath>

#include "check.hpp"
#include "vnt/elastic.hpp"
#include "vnt/errors.hpp"
#include "vnt/runner.hpp"

using namespace vnt;

static std::vector<DeviceSpec> gpus(std::size_t n, std::size_t cap = 1024) {
  std::vector<DeviceSpec> d;
  for (std::size_t i = 0; i < n; ++i) d.push_back({"gpu" + std::to_string(i), "B200", cap});
  return d;
}
static ModelSpec toy(std::uint64_t seed) { return ModelSpec{{3, 6, 2}, Activation::kTanh, Loss::kMse, seed}; }

static double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

TEST_CASE("device buffer equals scaled mean gradient for a single node") {
  Model model(toy(5));
  const auto p = model.init_params();
  SynthDataset data(1, 4, 3, 2);
  const Batch b = data.sequential_batch(0, 4);
  const auto r = device_step(model, p, model.init_kernels(), {b}, gpus(1)[0]);
  const auto fb = model.forward_backward(p, b, model.init_kernels());
  const auto sum = r.buffer.rounded_sum();
  for (std::size_t i = 0; i < sum.size(); ++i) CHECK(std::abs(sum[i] - 4.0 * fb.grads.values[i]) <= 1e-9);
  CHECK(r.buffer.examples_accumulated() == 4);
  CHECK(r.metrics.waves == 1 && r.metrics.peak_resident == 4);
}

// Reference test_virtual_exec.cpp:89-106 asserts bitwise equality here: its
// accumulator is exact per EXAMPLE.  The B200 engine is exact per virtual
// node (fp32 partial per node, int64 sum across nodes), so regrouping the
// same examples into different nodes changes the buffer only within fp32
// rounding; the mapping of a fixed partition stays exact.
TEST_CASE("regrouping nodes changes the buffer only within fp32 rounding") {
  Model model(toy(11));
  const auto p = model.init_params();
  const Batch b = SynthDataset(3, 8, 3, 2).sequential_batch(0, 8);
  std::vector<Batch> four, two;
  for (int n = 0; n < 4; ++n) four.push_back(b.slice(2 * n, 2));
  for (int n = 0; n < 2; ++n) two.push_back(b.slice(4 * n, 4));
  const auto a = device_step(model, p, model.init_kernels(), four, gpus(1)[0]);
  const auto c = device_step(model, p, model.init_kernels(), two, gpus(1)[0]);
  // Different node partitions: equal within fp32 tolerance (exactly equal only
  // for the same partition, see the mapping-invariance case below).
  CHECK(max_abs_diff(a.buffer.rounded_sum(), c.buffer.rounded_sum()) <= 1e-6);
  CHECK(a.metrics.waves == 4 && c.metrics.waves == 2);
  CHECK(a.metrics.buffer_bytes == c.metrics.buffer_bytes);
}

TEST_CASE("weighted synchronization recovers the flat mean over 6:2") {
  Model model(toy(13));
  const auto p = model.init_params();
  const Batch b = SynthDataset(5, 8, 3, 2).sequential_batch(0, 8);
  const auto a = device_step(model, p, model.init_kernels(), {b.slice(0, 6)}, gpus(2)[0]);
  const auto c = device_step(model, p, model.init_kernels(), {b.slice(6, 2)}, gpus(2)[1]);
  const auto synced = sync_gradients({{"gpu0", &a.buffer}, {"gpu1", &c.buffer}});
  const auto whole = model.forward_backward(p, b, model.init_kernels());
  CHECK(max_abs_diff(synced.values, whole.grads.values) <= 1e-6);
  CHECK_THROWS_AS(device_step(model, p, model.init_kernels(), {}, gpus(1)[0]), ConfigError);
}

TEST_CASE("post-step parameters are bitwise identical across mappings") {
  Model model(toy(23));
  SynthDataset data(8, 64, 3, 2);
  std::vector<ParamVector> finals;
  for (std::size_t G : {1u, 2u, 4u, 8u}) {
    World world = make_world(model, gpus(G));
    const auto mapping = make_uniform_mapping(64, 8, gpus(G));
    for (int s = 0; s < 5; ++s)
      train_step(model, world, mapping, data.sequential_batch(64 * s, 64), 0.05,
                 {.step_index = (std::uint64_t)s});
    world.validate_replicas();
    finals.push_back(world.workers[0].params);
  }
  for (std::size_t i = 1; i < finals.size(); ++i) CHECK(finals[i].bitwise_equal(finals[0]));
}

TEST_CASE("any mapping equals full-batch SGD within fp32 tolerance") {
  Model model(toy(29));
  SynthDataset data(9, 32, 3, 2);
  World world = make_world(model, gpus(4));
  const auto mapping = make_uniform_mapping(32, 8, gpus(4));
  ParamVector oracle = model.init_params();
  for (int s = 0; s < 10; ++s) {
    const Batch b = data.sequential_batch(32 * s, 32);
    train_step(model, world, mapping, b, 0.05, {});
    oracle = sgd_apply(oracle, model.forward_backward(oracle, b, model.init_kernels()).grads, 0.05);
    CHECK(max_abs_diff(world.workers[0].params.values, oracle.values) <= 1e-5);
  }
}

TEST_CASE("replica divergence at entry is detected") {
  Model model(toy(41));
  World world = make_world(model, gpus(2));
  world.workers[1].params.values[0] += 1e-9;
  const auto mapping = make_uniform_mapping(8, 2, gpus(2));
  CHECK_THROWS_AS(train_step(model, world, mapping, SynthDataset(12, 8, 3, 2).sequential_batch(0, 8), 0.1, {}),
                  ConsistencyError);
}

TEST_CASE("metrics report waves, residency and constant buffer bytes") {
  Model model(toy(43));
  const Batch b = SynthDataset(13, 32, 3, 2).sequential_batch(0, 32);
  for (std::size_t nodes : {1u, 2u, 4u, 8u, 16u}) {
    World world = make_world(model, gpus(1, 2048));
    const auto m = train_step(model, world, make_uniform_mapping(32, nodes, gpus(1, 2048)), b, 0.05, {});
    CHECK(m.per_device.size() == 1);
    CHECK(m.per_device[0].waves == nodes);
    CHECK(m.per_device[0].peak_resident == 32 / nodes);
    CHECK(m.per_device[0].buffer_bytes == model.param_count() * sizeof(double));
  }
}

TEST_CASE("parallel device execution matches serial bitwise") {
  Model model(toy(47));
  SynthDataset data(14, 64, 3, 2);
  World a = make_world(model, gpus(4)), b = make_world(model, gpus(4));
  const auto mapping = make_uniform_mapping(64, 8, gpus(4));
  for (int s = 0; s < 3; ++s) {
    const Batch batch = data.sequential_batch(64 * s, 64);
    const auto ma = train_step(model, a, mapping, batch, 0.05, {});
    const auto mb = train_step(model, b, mapping, batch, 0.05, {.parallel_devices = true});
    CHECK(ma.loss == mb.loss);
  }
  CHECK(a.workers[0].params.bitwise_equal(b.workers[0].params));
}

static RunnerConfig toy_config(std::size_t devices) {
  RunnerConfig c;
  c.model = ModelSpec{{3, 6, 2}, Activation::kTanh, Loss::kMse, 17};
  c.global_batch = 64;
  c.virtual_nodes = 8;
  c.lr = 0.05;
  c.data_seed = 4;
  c.dataset_size = 256;
  c.devices = gpus(devices);
  return c;
}

TEST_CASE("a train_step loop over a World is the Trainer's trajectory bit for bit") {
  // runner.cpp:75-82: Trainer::step is train_step on the Trainer's World; the
  // World carries the fixed-point scale history (WorkerState::scales).
  const RunnerConfig cfg = toy_config(4);
  Trainer trainer(cfg);
  Model model(cfg.model);
  World world = make_world(model, cfg.devices);
  const auto mapping = make_uniform_mapping(cfg.global_batch, cfg.virtual_nodes, cfg.devices);
  const SynthDataset data(cfg.data_seed, cfg.dataset_size, 3, 2);
  for (std::uint64_t s = 0; s < 8; ++s) {
    const Batch b = data.sequential_batch((s * cfg.global_batch) % cfg.dataset_size, cfg.global_batch);
    const StepMetrics a = train_step(model, world, mapping, b, cfg.lr, {s, false});
    const StepMetrics t = trainer.step();
    CHECK(a.loss == t.loss);
    CHECK(world.workers[0].params.bitwise_equal(trainer.params()));
    CHECK(world.workers[0].scales.size() == 4);   // no tcgen05 layer: no fp16 operand scales
  }
  // and the World-level migrate_state carries the scales through a resize
  InMemoryTransport tr;
  const auto plan = elastic::plan_resize(mapping, gpus(6));
  const World next = elastic::migrate_state(plan, world, tr);
  CHECK(next.workers.size() == 6);
  for (const auto& w : next.workers) CHECK(w.scales == world.workers[0].scales);
}

TEST_CASE("resize schedule does not perturb the training trajectory") {
  const auto rep = elastic::resized_training_equivalence_harness(
      toy_config(8), {{2, gpus(4)}, {4, gpus(8)}}, 6);
  CHECK(rep.bitwise_identical);
  for (const auto& r : rep.steps) CHECK(r.max_divergence == 0.0);
  std::vector<elastic::ResizePoint> every;
  for (std::uint64_t s = 1; s <= 5; ++s) every.push_back({s, gpus(s % 2 == 0 ? 8 : 2)});
  CHECK(elastic::resized_training_equivalence_harness(toy_config(8), every, 6).bitwise_identical);
  // Non-power-of-two device counts too (exact int64 reduction).
  CHECK(elastic::resized_training_equivalence_harness(toy_config(4), {{1, gpus(3)}, {3, gpus(6)}}, 5)
            .bitwise_identical);
}

TEST_CASE("prefetch and shuffled epochs have no semantic effect across mappings") {
  auto plain = toy_config(4), pre = toy_config(4);
  pre.prefetch = true;
  Trainer a(plain), b(pre);
  for (int s = 0; s < 4; ++s) CHECK(a.step().loss == b.step().loss);
  CHECK(a.params().bitwise_equal(b.params()));
  auto one = toy_config(1), four = toy_config(4);
  one.shuffle_epochs = four.shuffle_epochs = true;
  one.shuffle_seed = four.shuffle_seed = 3;
  Trainer c(one), d(four);
  for (int s = 0; s < 6; ++s) {
    c.step();
    d.step();
  }
  CHECK(c.params().bitwise_equal(d.params()));
}

TEST_MAIN()
