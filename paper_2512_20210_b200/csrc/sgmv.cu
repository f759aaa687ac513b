// Paged multi-LoRA prefill op (gathered SGMV, tcgen05) — see include/plora.h.
#include "plan.hpp"

using namespace plora;

extern "C" int plora_sgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream) {
  return guard([&]() -> int {
    throw std::logic_error("plora_sgmv: the tcgen05 prefill path is not built yet");
  });
}
