// C ABI of include/hrt_b200.h over the per-dtype engines.
#include <cstring>
#include <memory>
#include <utility>

#include "engine_iface.h"


// ===========================================================================
// C ABI
// ===========================================================================
using namespace hrtcore;

struct hrt_engine {
  std::unique_ptr<EngineBase> impl;
};

// per host thread: engines driven from several threads (EnginePool) must not race on it
static thread_local std::string g_last_error;

// need_eng: the call operates on an engine, so a NULL handle is an argument error
// (HRT_ERR_INVALID) rather than a dereference
template <class Fn>
static hrt_status guarded(hrt_engine* eng, bool need_eng, Fn&& fn) {
  try {
    if (!eng && need_eng) throw HrtError(HRT_ERR_INVALID, "null engine");
    if (eng) CUDA_OK(cudaSetDevice(eng->impl->device));
    fn();
    return HRT_OK;
  } catch (const HrtError& e) {
    if (eng) eng->impl->last_error = e.what();
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (eng) eng->impl->last_error = e.what();
    g_last_error = e.what();
    return HRT_ERR_CUDA;
  }
}
template <class Fn>
static hrt_status guarded(hrt_engine* eng, Fn&& fn) {
  return guarded(eng, true, std::forward<Fn>(fn));
}

extern "C" {

int64_t hrt_param_count(const hrt_config* cfg) { return engine_param_count(*cfg); }

hrt_status hrt_create(const hrt_config* cfg, const float* params, int64_t n_params, int32_t device, hrt_engine** out) {
  return guarded(nullptr, /*need_eng=*/false, [&] {
    if (!cfg || !params || !out) throw HrtError(HRT_ERR_INVALID, "null argument");
    if (n_params != engine_param_count(*cfg))
      throw HrtError(HRT_ERR_INVALID, "n_params " + std::to_string(n_params) + " != expected " +
                                          std::to_string(engine_param_count(*cfg)));
    auto e = std::make_unique<hrt_engine>();
    if (cfg->dtype == HRT_DTYPE_F32)
      e->impl.reset(new_engine_f32(*cfg, params, device));
    else if (cfg->dtype == HRT_DTYPE_BF16)
      e->impl.reset(new_engine_bf16(*cfg, params, device));
    else
      throw HrtError(HRT_ERR_INVALID, "unknown dtype");
    *out = e.release();
  });
}

void hrt_destroy(hrt_engine* eng) { delete eng; }

hrt_status hrt_estimate_arena(const hrt_config* cfg, int64_t* phase_bytes) {
  return guarded(nullptr, /*need_eng=*/false, [&] {
    if (!cfg || !phase_bytes) throw HrtError(HRT_ERR_INVALID, "null argument");
    if (cfg->dtype == HRT_DTYPE_F32)
      estimate_arena_f32(*cfg, phase_bytes);
    else if (cfg->dtype == HRT_DTYPE_BF16)
      estimate_arena_bf16(*cfg, phase_bytes);
    else
      throw HrtError(HRT_ERR_INVALID, "unknown dtype");
  });
}

const char* hrt_last_error(const hrt_engine* eng) {
  return eng ? eng->impl->last_error.c_str() : g_last_error.c_str();
}

hrt_status hrt_get_stats(const hrt_engine* eng, hrt_stats* out) {
  if (!eng || !out) return HRT_ERR_INVALID;
  *out = eng->impl->stats;
  return HRT_OK;
}

void* hrt_stream(hrt_engine* eng) { return eng ? (void*)eng->impl->stream : nullptr; }

hrt_status hrt_synchronize(hrt_engine* eng) {
  return guarded(eng, [&] { CUDA_OK(cudaStreamSynchronize(eng->impl->stream)); });
}

hrt_status hrt_encode(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t n_seq, float* memory_out) {
  return guarded(eng, [&] { eng->impl->encode(ids, lens, n_seq, memory_out); });
}

hrt_status hrt_start_cache(hrt_engine* eng, int32_t rows, int32_t cap, const int32_t* row_seq) {
  return guarded(eng, [&] { eng->impl->start_cache(rows, cap, row_seq); });
}

hrt_status hrt_step(hrt_engine* eng, const int32_t* tokens, int32_t position, float* logp_out) {
  return guarded(eng, [&] { eng->impl->step(tokens, position, logp_out); });
}

hrt_status hrt_reorder(hrt_engine* eng, const int32_t* parents) {
  return guarded(eng, [&] { eng->impl->reorder(parents); });
}

hrt_status hrt_parallel_logits(hrt_engine* eng, const int32_t* ids, const int32_t* positions, const uint8_t* pad_mask,
                               int32_t B, int32_t T, int32_t mode, const int32_t* seq, float* logits_out) {
  return guarded(eng, [&] { eng->impl->parallel_logits(ids, positions, pad_mask, B, T, mode, seq, logits_out); });
}

hrt_status hrt_argmax_logprobs(hrt_engine* eng, const int32_t* exclude, int32_t n_exclude, int32_t* amax_out,
                               float* lp_out) {
  return guarded(eng, [&] { eng->impl->argmax_logprobs(exclude, n_exclude, amax_out, lp_out); });
}

hrt_status hrt_translate_batch(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t B, int32_t k,
                               int32_t b_at, int32_t b_nat, float length_penalty, const int32_t* max_steps,
                               const hrt_translate_out* out, int32_t io_on_device) {
  return guarded(eng, [&] {
    if (!ids || !lens || !out) throw HrtError(HRT_ERR_INVALID, "null argument");
    eng->impl->translate(ids, lens, B, k, b_at, b_nat, length_penalty, max_steps, out, io_on_device, false);
  });
}

hrt_status hrt_at_translate_batch(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t B, int32_t beam,
                                  float length_penalty, const int32_t* max_steps, const hrt_translate_out* out,
                                  int32_t io_on_device) {
  return guarded(eng, [&] {
    if (!ids || !lens || !out) throw HrtError(HRT_ERR_INVALID, "null argument");
    eng->impl->translate(ids, lens, B, 1, beam, 1, length_penalty, max_steps, out, io_on_device, true);
  });
}

hrt_status hrt_set_option(hrt_engine* eng, const char* name, int32_t value) {
  return guarded(eng, [&] { eng->impl->set_option(name ? name : "", value); });
}

hrt_status hrt_phase_times(hrt_engine* eng, float* ms3) {
  return guarded(eng, [&] {
    EngineBase* e = eng->impl.get();
    if (!ms3) throw HrtError(HRT_ERR_INVALID, "null argument");
    if (!e->phase_valid) throw HrtError(HRT_ERR_INVALID, "no fused call recorded yet");
    CUDA_OK(cudaEventSynchronize(e->phase_ev[3]));
    for (int i = 0; i < 3; ++i) CUDA_OK(cudaEventElapsedTime(&ms3[i], e->phase_ev[i], e->phase_ev[i + 1]));
  });
}

hrt_status hrt_timing_enable(hrt_engine* eng, const char* kernel_class, int32_t enable) {
  return guarded(eng, [&] {
    EngineBase* e = eng->impl.get();
    int cls = 0;
    std::string c = kernel_class ? kernel_class : "all";
    if (c == "vocab") cls = K_VOCAB;
    else if (c == "gemm") cls = K_GEMM;
    else if (c == "attn") cls = K_ATTN;
    else if (c == "all") cls = K_GEMM | K_VOCAB | K_ATTN | K_OTHER;
    else throw HrtError(HRT_ERR_INVALID, "unknown kernel class " + c);
    CUDA_OK(cudaStreamSynchronize(e->stream));
    e->timed_class = enable ? cls : 0;
    e->ev_used = 0;
    e->t_bytes = e->t_flops = 0;
    e->t_launches = 0;
  });
}

hrt_status hrt_timing_report(hrt_engine* eng, char* buf, int64_t cap) {
  return guarded(eng, [&] {
    EngineBase* e = eng->impl.get();
    CUDA_OK(cudaStreamSynchronize(e->stream));
    struct Agg {
      double ms = 0, flops = 0;
      int n = 0;
    };
    std::map<std::string, Agg> agg;
    for (size_t i = 0; i < e->ev_used; ++i) {
      float m = 0;
      CUDA_OK(cudaEventElapsedTime(&m, e->ev_pool[i].first, e->ev_pool[i].second));
      Agg& a = agg[e->ev_tag[i] ? e->ev_tag[i] : "untagged"];
      a.ms += m;
      a.n += 1;
      a.flops += e->ev_flops[i];
    }
    std::string s = "{";
    for (auto& kv : agg) {
      if (s.size() > 1) s += ", ";
      s += "\"" + kv.first + "\": [" + std::to_string(kv.second.ms) + ", " + std::to_string(kv.second.n) + ", " +
           std::to_string(kv.second.flops) + "]";
    }
    s += "}";
    if (!buf || (int64_t)s.size() + 1 > cap) throw HrtError(HRT_ERR_INVALID, "report buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

hrt_status hrt_timing_read(hrt_engine* eng, double* total_ms, int64_t* launches, double* alg_bytes,
                           double* alg_flops) {
  return guarded(eng, [&] {
    EngineBase* e = eng->impl.get();
    CUDA_OK(cudaStreamSynchronize(e->stream));
    double ms = 0;
    for (size_t i = 0; i < e->ev_used; ++i) {
      float m = 0;
      CUDA_OK(cudaEventElapsedTime(&m, e->ev_pool[i].first, e->ev_pool[i].second));
      ms += m;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = e->t_launches;
    if (alg_bytes) *alg_bytes = e->t_bytes;
    if (alg_flops) *alg_flops = e->t_flops;
  });
}

}  // extern "C"
