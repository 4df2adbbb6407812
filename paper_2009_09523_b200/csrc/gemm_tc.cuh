// tcgen05 / TMA tensor-core path (filled in below the FFMA baseline).
#pragma once

namespace {
bool tc_layer_eligible(int, uint64_t, uint64_t) { return false; }
void tc_init(vnt_engine*) {}
void tc_destroy(vnt_engine*) {}
void tc_forward(vnt_engine*, int, int, int, const int*, bool) {
  throw vntb::EngineError(1, "tcgen05 path not built");
}
void tc_weight_grad(vnt_engine*, int, const Pass&, const int*, const int*, float, float, bool, int) {
  throw vntb::EngineError(1, "tcgen05 path not built");
}
void tc_backward_data(vnt_engine*, int, int, int, const int*) {
  throw vntb::EngineError(1, "tcgen05 path not built");
}
}  // namespace
