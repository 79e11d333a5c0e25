// fp32 engine instantiation (C1 parity config): SIMT / GEMV fp32 kernels.
// The kernel namespace is renamed per translation unit so the two dtype TUs
// can be compiled in parallel and linked without duplicate kernel symbols.
#define hrt hrt_f32
#include "engine.cuh"

namespace hrtcore {
EngineBase* new_engine_f32(const hrt_config& c, const float* params, int dev) {
  return new hrt_f32::Engine<float>(c, params, dev);
}
void estimate_arena_f32(const hrt_config& c, int64_t* phase_bytes) {
  hrt_f32::Engine<float>::estimate(c, phase_bytes);
}
int64_t engine_param_count(const hrt_config& c) { return hrt_f32::Engine<float>::param_count(c); }
}  // namespace hrtcore
