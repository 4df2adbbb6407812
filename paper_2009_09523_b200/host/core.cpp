// vnt drop-in: errors, RNG, batches, synthetic data, exact sums (host side).
// Semantics follow the reference (rng.cpp, data.cpp, exact_sum.hpp in
// /root/reference/proj/core); bit-identity is tested against the oracle.
#include <cmath>
#include <numbers>
#include <unordered_set>

#include "vnt/data.hpp"
#include "vnt/errors.hpp"
#include "vnt/exact_sum.hpp"
#include "vnt/rng.hpp"
#include "vnt_engine.h"

namespace vnt {

void raise_status(int status, const std::string& context) {
  if (status == VNT_OK) return;
  const std::string msg = context + ": " + vnt_last_error();
  switch (status) {
    case VNT_ERR_CONFIG: throw ConfigError(msg);
    case VNT_ERR_CAPACITY: throw CapacityError(msg);
    case VNT_ERR_SHAPE: throw ShapeError(msg);
    case VNT_ERR_CONSISTENCY: throw ConsistencyError(msg);
    case VNT_ERR_MIGRATION: throw MigrationError(msg);
    default: throw Error(msg);
  }
}

// ------------------------------------------------------------------- RNG
namespace {
constexpr std::uint64_t kPhi = 0x9E3779B97F4A7C15ULL;

std::uint64_t finalize(std::uint64_t z) {  // splitmix64 output function
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

std::uint64_t label_hash(std::string_view s) {  // FNV-1a 64
  std::uint64_t h = 0xCBF29CE484222325ULL;
  for (unsigned char c : s) h = (h ^ c) * 0x100000001B3ULL;
  return h;
}
}  // namespace

CounterRng::CounterRng(std::uint64_t seed) : key_(finalize(seed + kPhi)) {}

CounterRng CounterRng::from_key(std::uint64_t key) {
  CounterRng r;
  r.key_ = key;
  return r;
}

CounterRng CounterRng::split(std::uint64_t stream) const {
  return from_key(finalize(key_ ^ finalize(stream + kPhi)));
}

CounterRng CounterRng::split(std::string_view label) const { return split(label_hash(label)); }

std::uint64_t CounterRng::bits(std::uint64_t counter) const { return finalize(key_ + counter * kPhi); }

double CounterRng::uniform(std::uint64_t counter) const {
  return static_cast<double>(bits(counter) >> 11) * 0x1.0p-53;
}

double CounterRng::normal(std::uint64_t counter) const {
  const double u1 = static_cast<double>((bits(2 * counter) >> 11) + 1) * 0x1.0p-53;  // (0,1]
  const double u2 = static_cast<double>(bits(2 * counter + 1) >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}

std::uint64_t CounterRng::below(std::uint64_t counter, std::uint64_t bound) const {
  if (bound == 0) throw ConfigError("CounterRng::below: bound must be positive");
  return bits(counter) % bound;
}

std::vector<std::uint64_t> random_permutation(const CounterRng& rng, std::uint64_t n) {
  std::vector<std::uint64_t> p(n);
  for (std::uint64_t i = 0; i < n; ++i) p[i] = i;
  for (std::uint64_t i = n; i > 1; --i) std::swap(p[i - 1], p[rng.below(i, i)]);
  return p;
}

// ----------------------------------------------------------------- Batch
void Batch::validate() const {
  if (count == 0) throw ConfigError("Batch: count must be >= 1");
  if (examples.size() != count * input_width)
    throw ShapeError("Batch: examples size does not match count x input_width");
  if (labels.size() != count * output_width)
    throw ShapeError("Batch: labels size does not match count x output_width");
  if (ids.size() != count) throw ShapeError("Batch: ids size does not match count");
  if (std::unordered_set<std::uint64_t>(ids.begin(), ids.end()).size() != ids.size())
    throw ConfigError("Batch: example ids must be distinct");
}

std::span<const double> Batch::example(std::size_t i) const {
  return {examples.data() + i * input_width, input_width};
}

std::span<const double> Batch::label(std::size_t i) const {
  return {labels.data() + i * output_width, output_width};
}

Batch Batch::slice(std::size_t begin, std::size_t len) const {
  if (begin + len > count) throw ConfigError("Batch::slice: out of range");
  Batch b;
  b.count = len;
  b.input_width = input_width;
  b.output_width = output_width;
  b.examples.assign(examples.begin() + begin * input_width,
                    examples.begin() + (begin + len) * input_width);
  b.labels.assign(labels.begin() + begin * output_width,
                  labels.begin() + (begin + len) * output_width);
  b.ids.assign(ids.begin() + begin, ids.begin() + begin + len);
  return b;
}

// ---------------------------------------------------------- SynthDataset
SynthDataset::SynthDataset(std::uint64_t seed, std::size_t n, std::size_t in, std::size_t out)
    : seed_(seed), n_(n), in_(in), out_(out) {
  if (n == 0 || in == 0 || out == 0) throw ConfigError("SynthDataset: sizes must be positive");
  const CounterRng t = CounterRng(seed).split("teacher");
  const double scale = 1.0 / std::sqrt(static_cast<double>(in));
  teacher_.resize(in * out);
  for (std::size_t k = 0; k < teacher_.size(); ++k) teacher_[k] = t.normal(k) * scale;
}

Batch SynthDataset::batch(std::span<const std::uint64_t> ids) const {
  Batch b;
  b.count = ids.size();
  b.input_width = in_;
  b.output_width = out_;
  b.examples.resize(b.count * in_);
  b.labels.resize(b.count * out_);
  b.ids.assign(ids.begin(), ids.end());
  const CounterRng xr = CounterRng(seed_).split("examples");
  std::vector<double> z(out_);
  for (std::size_t r = 0; r < ids.size(); ++r) {
    const std::uint64_t id = ids[r];
    if (id >= n_) throw ConfigError("SynthDataset: example id out of range");
    double* x = b.examples.data() + r * in_;
    for (std::size_t j = 0; j < in_; ++j) x[j] = xr.normal(id * in_ + j);
    double top = -1e300;
    for (std::size_t o = 0; o < out_; ++o) {
      double acc = 0.0;
      for (std::size_t j = 0; j < in_; ++j) acc += x[j] * teacher_[j * out_ + o];
      z[o] = acc;
      top = std::max(top, acc);
    }
    double norm = 0.0;
    for (std::size_t o = 0; o < out_; ++o) {
      z[o] = std::exp(z[o] - top);
      norm += z[o];
    }
    for (std::size_t o = 0; o < out_; ++o) b.labels[r * out_ + o] = z[o] / norm;
  }
  b.validate();
  return b;
}

Batch SynthDataset::sequential_batch(std::uint64_t start, std::size_t count) const {
  std::vector<std::uint64_t> ids(count);
  for (std::size_t i = 0; i < count; ++i) ids[i] = (start + i) % n_;
  return batch(ids);
}

SynthDataset synth_dataset(std::uint64_t seed, std::size_t n, std::size_t in, std::size_t out) {
  return SynthDataset(seed, n, in, out);
}

// ------------------------------------------------------------ exact sums
// Non-overlapping expansion (Shewchuk grow-expansion); total() rounds once.
void ExactAccumulator::add(double x) {
  if (x == 0.0) return;
  if (!std::isfinite(x)) throw Error("ExactAccumulator: non-finite value");
  std::size_t keep = 0;
  for (double y : parts_) {
    if (std::fabs(x) < std::fabs(y)) std::swap(x, y);
    const double hi = x + y;
    const double lo = y - (hi - x);
    if (lo != 0.0) parts_[keep++] = lo;
    x = hi;
  }
  parts_.resize(keep);
  parts_.push_back(x);
}

void ExactAccumulator::merge(const ExactAccumulator& other) {
  for (double p : other.parts_) add(p);
}

double ExactAccumulator::total() const {
  std::size_t n = parts_.size();
  if (n == 0) return 0.0;
  double hi = parts_[--n], lo = 0.0;
  while (n > 0) {
    const double x = hi, y = parts_[--n];
    hi = x + y;
    lo = y - (hi - x);
    if (lo != 0.0) break;
  }
  if (n > 0 && ((lo < 0.0 && parts_[n - 1] < 0.0) || (lo > 0.0 && parts_[n - 1] > 0.0))) {
    const double y = lo * 2.0, x = hi + y;
    if (y == x - hi) hi = x;
  }
  return hi;
}

void ExactVectorAccumulator::add(std::span<const double> values) {
  if (values.size() != elems_.size()) throw ShapeError("ExactVectorAccumulator: size mismatch");
  for (std::size_t i = 0; i < values.size(); ++i) elems_[i].add(values[i]);
}

void ExactVectorAccumulator::merge(const ExactVectorAccumulator& other) {
  if (other.elems_.size() != elems_.size())
    throw ShapeError("ExactVectorAccumulator: size mismatch");
  for (std::size_t i = 0; i < elems_.size(); ++i) elems_[i].merge(other.elems_[i]);
}

std::vector<double> ExactVectorAccumulator::rounded() const {
  std::vector<double> out(elems_.size());
  for (std::size_t i = 0; i < elems_.size(); ++i) out[i] = elems_[i].total();
  return out;
}

void ExactVectorAccumulator::reset() {
  for (auto& e : elems_) e.reset();
}

}  // namespace vnt
