// bf16 engine instantiation (C2-C5): tcgen05 GEMMs, mma.sync GEMV / attention.
#define hrt hrt_bf16
#include "engine.cuh"

namespace hrtcore {
EngineBase* new_engine_bf16(const hrt_config& c, const float* params, int dev) {
  return new hrt_bf16::Engine<hrt_bf16::bf16>(c, params, dev);
}
void estimate_arena_bf16(const hrt_config& c, int64_t* phase_bytes) {
  hrt_bf16::Engine<hrt_bf16::bf16>::estimate(c, phase_bytes);
}
}  // namespace hrtcore
