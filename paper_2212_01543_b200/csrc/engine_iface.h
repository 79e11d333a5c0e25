// Engine interface shared by the per-dtype translation units and the C ABI
// (engine_f32.cu / engine_bf16.cu instantiate Engine<T>; capi.cu exports
// include/hrt_b200.h). Kept free of kernel headers so it compiles anywhere.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hrt_b200.h"

namespace hrtcore {

struct HrtError : std::runtime_error {
  hrt_status code;
  HrtError(hrt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t _e = (x);                                                                              \
    if (_e != cudaSuccess)                                                                             \
      throw HrtError(HRT_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e) + " @" + \
                                       std::to_string(__LINE__));                                      \
  } while (0)

static inline int cdiv(int a, int b) { return (a + b - 1) / b; }
static inline size_t align_up(size_t n, size_t a = 256) { return (n + a - 1) / a * a; }

enum KClass { K_GEMM = 1, K_VOCAB = 2, K_ATTN = 4, K_OTHER = 8 };


// ---------------------------------------------------------------------------
// engine
// ---------------------------------------------------------------------------
struct EngineBase {
  hrt_config cfg{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string last_error;
  hrt_stats stats{};
  // phase timing: events at the phase boundaries of the last fused call
  cudaEvent_t phase_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool phase_valid = false;
  void phase_mark(int i) {
    if (!phase_ev[i]) cudaEventCreate(&phase_ev[i]);
    cudaEventRecord(phase_ev[i], stream);
  }
  // kernel-class timing
  int timed_class = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  std::vector<const char*> ev_tag;
  std::vector<double> ev_flops;  // algorithmic FLOPs of each timed launch
  size_t ev_used = 0;
  const char* cur_tag = "untagged";  // call-site tag for the next launches
  double t_bytes = 0, t_flops = 0;
  int64_t t_launches = 0;

  virtual ~EngineBase() {
    for (auto& p : ev_pool) {
      cudaEventDestroy(p.first);
      cudaEventDestroy(p.second);
    }
    if (stream) cudaStreamDestroy(stream);
  }
  virtual void encode(const int32_t* ids, const int32_t* lens, int n, float* mem_out) = 0;
  virtual void start_cache(int rows, int cap, const int32_t* row_seq) = 0;
  virtual void step(const int32_t* tokens, int position, float* logp_out) = 0;
  virtual void reorder(const int32_t* parents) = 0;
  virtual void parallel_logits(const int32_t* ids, const int32_t* pos, const uint8_t* pad, int B, int T, int mode,
                               const int32_t* seq, float* logits_out) = 0;
  virtual void argmax_logprobs(const int32_t* excl, int n_excl, int32_t* amax, float* lp) = 0;
  virtual void set_option(const std::string& name, int value) = 0;
  virtual void translate(const int32_t* ids, const int32_t* lens, int B, int k, int b_at, int b_nat, float alpha,
                         const int32_t* caps, const hrt_translate_out* out, int on_device, bool at) = 0;

  // --- launch bookkeeping -------------------------------------------------
  struct Scope {
    EngineBase* e;
    std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
    Scope(EngineBase* eng, int cls, double bytes, double flops) : e(eng) {
      if (e->timed_class & cls) {
        if (e->ev_used == e->ev_pool.size()) {
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          e->ev_pool.emplace_back(a, b);
        }
        if (e->ev_tag.size() < e->ev_pool.size()) e->ev_tag.resize(e->ev_pool.size());
        if (e->ev_flops.size() < e->ev_pool.size()) e->ev_flops.resize(e->ev_pool.size());
        e->ev_tag[e->ev_used] = e->cur_tag;
        e->ev_flops[e->ev_used] = flops;
        ev = &e->ev_pool[e->ev_used++];
        cudaEventRecord(ev->first, e->stream);
        e->t_bytes += bytes;
        e->t_flops += flops;
        e->t_launches += 1;
      }
    }
    ~Scope() {
      if (ev) cudaEventRecord(ev->second, e->stream);
      e->stats.kernel_launches += 1;
    }
  };
  bool pdl = true;  // programmatic dependent launch on every kernel
  // dynamic shared-memory opt-in: cudaFuncSetAttribute is per device context,
  // so the cache is keyed on (device, kernel) and guarded for engines driven
  // from several host threads
  template <class K>
  void smem_optin(K kern, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[std::make_pair(device, reinterpret_cast<const void*>(kern))];
    if (have >= bytes) return;
    CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
  }
  int launch_cluster = 1;  // cluster size of the next launch (set by tc_launch only)
  template <typename... KArgs, typename... Args>
  void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (launch_cluster > 1) {  // thread-block clusters along x (tcgen05 GEMM CTA pairs)
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = launch_cluster;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t er = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (er != cudaSuccess) {
      const char* fname = nullptr;
      if (cudaFuncGetName(&fname, reinterpret_cast<const void*>(kern)) != cudaSuccess) fname = "?";
      throw HrtError(HRT_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(er) + " (" + fname + ", grid " +
                                       std::to_string(grid.x) + "x" + std::to_string(grid.y) + ", block " +
                                       std::to_string(block.x) + ", smem " + std::to_string(smem) + ", cluster " +
                                       std::to_string(launch_cluster) + ")");
    }
  }
  struct Tag {
    EngineBase* e;
    const char* prev;
    Tag(EngineBase* eng, const char* t) : e(eng), prev(eng->cur_tag) { e->cur_tag = t; }
    ~Tag() { e->cur_tag = prev; }
  };
  void check_launch() {
    cudaError_t er = cudaGetLastError();
    if (er != cudaSuccess) throw HrtError(HRT_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(er));
  }
};

// per-dtype factories (engine_f32.cu, engine_bf16.cu)
EngineBase* new_engine_f32(const hrt_config& c, const float* params, int dev);
EngineBase* new_engine_bf16(const hrt_config& c, const float* params, int dev);
int64_t engine_param_count(const hrt_config& c);
void estimate_arena_f32(const hrt_config& c, int64_t* phase_bytes);
void estimate_arena_bf16(const hrt_config& c, int64_t* phase_bytes);

}  // namespace hrtcore
