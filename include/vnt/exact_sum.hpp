// vnt drop-in: exact fp64 accumulation (reference exact_sum.hpp:34-69).
// Host-side; the GPU path reduces gradients exactly in int64 fixed point
// and these types only carry results across the API.
// Implementation: non-overlapping expansions (Shewchuk) with one correct
// rounding — same rounded result as the reference's limb accumulator.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

namespace vnt {

class ExactAccumulator {
 public:
  void add(double value);
  void merge(const ExactAccumulator& other);
  double total() const;
  void reset() { parts_.clear(); }

 private:
  std::vector<double> parts_;
};

class ExactVectorAccumulator {
 public:
  explicit ExactVectorAccumulator(std::size_t size) : elems_(size) {}
  std::size_t size() const { return elems_.size(); }
  void add(std::span<const double> values);
  void merge(const ExactVectorAccumulator& other);
  std::vector<double> rounded() const;
  void reset();

 private:
  std::vector<ExactAccumulator> elems_;
};

}  // namespace vnt
