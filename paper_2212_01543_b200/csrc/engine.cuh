// B200-native HRT inference engine: weights, device arena, the three phases
// (encoder, Stage-I skip-AT, Stage-II fill), and the C ABI of include/hrt_b200.h.
//
// Reference path (/root/reference/pkg/src/hrt): infer.py (session), decoding.py
// (search/selection), arena.py (buffer reuse), kernels.py (LN/softmax).
// Batched execution reproduces per-sentence results: sentences are packed
// ("varlen") so no padded key is ever attended; Stage-I rows of different
// sentences are independent; Stage-II candidates own disjoint row slots.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hrt_b200.h"
#include "common.cuh"
#include "gemm_epi.cuh"
#include "gemm_simt.cuh"
#include "gemv_small.cuh"
#include "kernels.cuh"
#include "tc_gemm.cuh"
#include "tc_gemm_ln.cuh"
#include "tc_gemm_lnrow.cuh"
#include "decode_cluster.cuh"
#include "tmap.h"

#include "engine_iface.h"

namespace hrt {
using namespace hrtcore;

// ---------------------------------------------------------------------------
// Device arena: one allocation, per-phase buffer plans carved at fixed
// offsets; phases alias each other (reference arena.py:23-51; LightSeq-style
// reuse). Sized once in closed form from the engine capacity.
// ---------------------------------------------------------------------------
struct Plan {
  size_t off = 0;
  template <typename X>
  X* take(char* base, size_t count) {
    size_t o = off;
    off = align_up(off + count * sizeof(X));
    return base ? reinterpret_cast<X*>(base + o) : nullptr;
  }
};


template <typename T>
struct Engine : EngineBase {
  static constexpr bool BF16 = std::is_same<T, bf16>::value;
  int d, ff, H, dh, Le, Ld, V, Lmax, P;  // P = PE rows
  float emb_scale, att_scale;

  // ---- weights ----
  struct EncW {
    T *wqkv, *wo, *w1, *w2;
    float *bqkv, *bo, *b1, *b2, *ln1g, *ln1b, *ln2g, *ln2b;
  };
  struct DecW {
    T *wqkv, *wo, *wqc, *woc, *w1, *w2;
    float *bqkv, *bo, *bqc, *boc, *b1, *b2, *ln1g, *ln1b, *ln2g, *ln2b, *ln3g, *ln3b;
  };
  std::vector<EncW> enc;
  std::vector<DecW> dec;
  T *E = nullptr, *wxkv = nullptr;
  float *bxkv = nullptr, *pe = nullptr, *enc_lng, *enc_lnb, *dec_lng, *dec_lnb;
  char* wblob = nullptr;
  char* vblob = nullptr;

  // ---- capacity ----
  int Bmax, beam_max, Me_max, R_max, cap_max, M2_max, Mm_max, nt_max, logit_rows;

  // ---- persistent device buffers ----
  char* persist = nullptr;
  int *d_ids_raw, *d_ids, *d_pos, *d_meta;
  T* xkv;  // [Me_max][Ld*2d]
  // Stage-I state
  int *s_feed, *s_done, *s_nsteps, *s_forced, *s_anchors, *s_caps, *s_hist, *s_hist2, *s_rowseq, *s_parents;
  double* s_score;
  // device beam search state (fused b_at > 1 path)
  int *b_greedy, *b_anchors2, *b_live, *b_nfin, *b_gdone, *b_fcount, *b_fgslot, *b_flist, *b_flen, *b_fforced,
      *b_ftok;
  double* b_fscore;
  int *c_off, *c_len, *c_forced;
  double* c_sat;
  StepCtl* s_ctl;
  int *s_alive, *s_srcoff, *s_srclen;
  // captured Stage-I loops (conditional WHILE graph), keyed by row bucket
  struct LoopGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int kernels = 0;
  };
  std::map<int, LoopGraph> loop_graphs;
  bool use_graphs = true;
  int attn_head_groups = 4;  // option "attn_head_groups": CTAs per (sequence, query block) in that kernel
  int attn_heads_mode = 1;  // option "attn_heads": all-heads-per-CTA prefill attention (0 off, 1 auto, 2 always)
  int attn_rows_mode = 1;  // option "attn_rows": CTA-per-row decode attention (0 off, 1 >= 256 rows, 2 always)
  // set in the fused Stage-I loop only: the encoder is complete (a stream copy separates
  // it from Stage I), so cross-attention K/V may be read before the PDL wait
  bool cross_prefetch = false;
  int debug_spin_us = 0;
  int enc_skip = 0;  // option "enc_skip" (debug attribution of the encoder kernels)  // option "debug_spin" (host-bound vs device-bound attribution)
  bool greedy_hist_identity = false;  // set during greedy Stage I: history map is the identity
  // debug: drop kernel groups from the Stage-I step (timing attribution only;
  // results are meaningless when nonzero). 1 LN, 2 attention, 4 GEMMs,
  // 8 vocab, 16 select, 32 embed.
  int s1_skip = 0;
  // outputs (device I/O staging)
  int *o_tokens, *o_lens, *o_calls;
  double* o_scores;
  unsigned char* o_forced;
  int* h_meta = nullptr;  // pinned staging for per-call metadata (one H2D copy)
  StepCtl* h_ctl = nullptr;  // pinned copy of the loop control after a call (row statistics)
  bool unrolled_last = false;
  char* h_out = nullptr;  // pinned staging for the packed per-call outputs (one D2H copy)
  size_t h_out_bytes = 0;
  int meta_cap;
  size_t meta_hdr = 0;     // ints reserved at the start for the fixed header
  cudaEvent_t meta_ev = nullptr;

  // ---- arena ----
  char* arena = nullptr;
  size_t arena_bytes = 0;
  struct EncBufs {
    float* x;
    T *y, *qkv, *ctx, *hid;
  } eb;
  struct S1Bufs {
    float* x;
    T *y, *qkv, *qc, *ctx, *hid, *kc, *vc;
    VocabParts parts;
    RowStat* rowstat;
    float* logits;
  } s1;
  struct S2Bufs {
    float* x;
    T *y, *qkv, *qc, *ctx, *hid, *ymask;
    int *ids, *pos, *out_row;
    VocabParts parts;
    RowStat* mstat;
    float* logits;
  } s2;

  // protocol-face state
  int p_rows = 0, p_cap = 0, p_len = 0, p_last_pos = -1, p_nseq = 0;
  bool p_has_cache = false;
  std::vector<int> p_seq_off, p_seq_len;  // encoded sequences (host copy)
  int p_B = 0, p_T = 0;
  float* p_logits = nullptr;  // [p_B*p_T][V] last parallel logits
  size_t p_logits_cap = 0;
  float* p_mem = nullptr;
  size_t p_mem_cap = 0;

  std::map<std::tuple<const void*, int, int, int, int>, CUtensorMap> tmaps;

  Engine(const hrt_config& c, const float* params, int dev) {
    cfg = c;
    device = dev;
    d = c.d_model;
    ff = c.d_ff;
    H = c.n_heads;
    dh = d / H;
    Le = c.enc_layers;
    Ld = c.dec_layers;
    V = c.vocab_size;
    Lmax = c.max_len;
    P = c.max_len + c.max_chunk + 1;
    emb_scale = (float)std::sqrt((double)d);
    att_scale = (float)(1.0 / std::sqrt((double)dh));
    if (d <= 0 || ff <= 0 || H <= 0 || d % H || Le < 0 || Ld < 1 || V < 8 || Lmax < 1 || c.max_chunk < 1)
      throw HrtError(HRT_ERR_INVALID, "invalid model shape");
    if (d > 1024) throw HrtError(HRT_ERR_INVALID, "d_model > 1024 unsupported");
    if (BF16 && (d % 64 || ff % 64))
      throw HrtError(HRT_ERR_INVALID, "bf16 engine needs d_model and d_ff multiples of 64 (tcgen05 K tiles)");
    CUDA_OK(cudaSetDevice(dev));
    CUDA_OK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_OK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (BF16 && V % 4) throw HrtError(HRT_ERR_INVALID, "bf16 engine needs vocab_size % 4 == 0");
    load_weights(params);
    size_capacity();
    alloc_buffers();
    CUDA_OK(cudaStreamSynchronize(stream));
  }

  ~Engine() override {
    cudaSetDevice(device);
    cudaFree(wblob);
    cudaFree(fblob);
    cudaFree(vblob);
    cudaFree(persist);
    cudaFree(arena);
    cudaFree(p_logits);
    cudaFree(p_mem);
    cudaFree(sk_ws);
    cudaFree(sk_counters);
    cudaFree(gv_counter);
    if (h_meta) cudaFreeHost(h_meta);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (h_out) cudaFreeHost(h_out);
    drop_loop_graphs();
    if (meta_ev) cudaEventDestroy(meta_ev);
  }

  // -------------------------------------------------------------------------
  // weights: fp32 blob in model.py:146-181 order -> transposed K-major T
  // matrices (QKV fused, all decoder cross-K/V fused) + fp32 vectors.
  // -------------------------------------------------------------------------
  void load_weights(const float* params) {
    const int64_t n = param_count(cfg);
    float* dsrc = nullptr;
    CUDA_OK(cudaMalloc(&dsrc, n * sizeof(float)));
    CUDA_OK(cudaMemcpy(dsrc, params, n * sizeof(float), cudaMemcpyHostToDevice));
    // matrix storage
    size_t mats = (size_t)V * d + (size_t)Le * (4 * d * d + 2 * d * ff) +
                  (size_t)Ld * (8 * d * d + 2 * d * ff);
    size_t vecs = (size_t)P * d + (size_t)Le * (4 * d + d + ff + d + 4 * d) + 2 * d +
                  (size_t)Ld * (3 * d + d + d + d + ff + d + 6 * d + 2 * d) + 2 * d + 64;
    CUDA_OK(cudaMalloc(&wblob, mats * sizeof(T) + 256));
    CUDA_OK(cudaMalloc(&vblob, vecs * sizeof(float) + 4096));
    stats.weight_bytes = (int64_t)(mats * sizeof(T) + vecs * sizeof(float));
    // Stage-I weights (vocabulary E, cross-K/V, decoder layers) are read every
    // decode step: they go first, contiguous, so one L2 persisting window
    // covers them; the encoder matrices (used once per batch) follow.
    hot_bytes = ((size_t)V * d + (size_t)Ld * (8 * d * d + 2 * d * ff)) * sizeof(T);
    T* wp_hot = reinterpret_cast<T*>(wblob);
    T* wp = wp_hot + (size_t)V * d + (size_t)Ld * (8 * d * d + 2 * d * ff);
    float* vp = reinterpret_cast<float*>(vblob);
    auto tmat = [&](size_t cnt) {
      T* r = wp;
      wp += cnt;
      return r;
    };
    auto tmat_hot = [&](size_t cnt) {
      T* r = wp_hot;
      wp_hot += cnt;
      return r;
    };
    auto tvec = [&](size_t cnt) {
      float* r = vp;
      vp += align_up(cnt, 16);
      return r;
    };
    int64_t off = 0;
    auto src = [&](int64_t cnt) {
      const float* r = dsrc + off;
      off += cnt;
      return r;
    };
    // transpose (K x N row-major fp32) -> (N x K) T rows of dst
    auto put_t = [&](const float* s, int K, int N, T* dst) {
      transpose_convert(s, K, N, dst);
    };
    auto put_v = [&](const float* s, int cnt, float* dst) {
      CUDA_OK(cudaMemcpyAsync(dst, s, cnt * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    };
    E = tmat_hot((size_t)V * d);
    convert(src((int64_t)V * d), (size_t)V * d, E);
    enc.resize(Le);
    for (int i = 0; i < Le; ++i) {
      EncW& w = enc[i];
      w.wqkv = tmat((size_t)3 * d * d);
      w.wo = tmat((size_t)d * d);
      w.w1 = tmat((size_t)ff * d);
      w.w2 = tmat((size_t)d * ff);
      w.bqkv = tvec(3 * d);
      w.bo = tvec(d);
      w.b1 = tvec(ff);
      w.b2 = tvec(d);
      w.ln1g = tvec(d);
      w.ln1b = tvec(d);
      w.ln2g = tvec(d);
      w.ln2b = tvec(d);
      put_v(src(d), d, w.ln1g);
      put_v(src(d), d, w.ln1b);
      put_t(src((int64_t)d * d), d, d, w.wqkv);
      put_t(src((int64_t)d * d), d, d, w.wqkv + (size_t)d * d);
      put_t(src((int64_t)d * d), d, d, w.wqkv + (size_t)2 * d * d);
      put_t(src((int64_t)d * d), d, d, w.wo);
      put_v(src(d), d, w.bqkv);
      put_v(src(d), d, w.bqkv + d);
      put_v(src(d), d, w.bqkv + 2 * d);
      put_v(src(d), d, w.bo);
      put_v(src(d), d, w.ln2g);
      put_v(src(d), d, w.ln2b);
      put_t(src((int64_t)d * ff), d, ff, w.w1);
      put_v(src(ff), ff, w.b1);
      put_t(src((int64_t)ff * d), ff, d, w.w2);
      put_v(src(d), d, w.b2);
    }
    enc_lng = tvec(d);
    enc_lnb = tvec(d);
    put_v(src(d), d, enc_lng);
    put_v(src(d), d, enc_lnb);
    dec.resize(Ld);
    wxkv = tmat_hot((size_t)Ld * 2 * d * d);
    bxkv = tvec((size_t)Ld * 2 * d);
    for (int i = 0; i < Ld; ++i) {
      DecW& w = dec[i];
      w.wqkv = tmat_hot((size_t)3 * d * d);
      w.wo = tmat_hot((size_t)d * d);
      w.wqc = tmat_hot((size_t)d * d);
      w.woc = tmat_hot((size_t)d * d);
      w.w1 = tmat_hot((size_t)ff * d);
      w.w2 = tmat_hot((size_t)d * ff);
      w.bqkv = tvec(3 * d);
      w.bo = tvec(d);
      w.bqc = tvec(d);
      w.boc = tvec(d);
      w.b1 = tvec(ff);
      w.b2 = tvec(d);
      w.ln1g = tvec(d);
      w.ln1b = tvec(d);
      w.ln2g = tvec(d);
      w.ln2b = tvec(d);
      w.ln3g = tvec(d);
      w.ln3b = tvec(d);
      put_v(src(d), d, w.ln1g);
      put_v(src(d), d, w.ln1b);
      put_t(src((int64_t)d * d), d, d, w.wqkv);
      put_t(src((int64_t)d * d), d, d, w.wqkv + (size_t)d * d);
      put_t(src((int64_t)d * d), d, d, w.wqkv + (size_t)2 * d * d);
      put_t(src((int64_t)d * d), d, d, w.wo);
      put_v(src(d), d, w.bqkv);
      put_v(src(d), d, w.bqkv + d);
      put_v(src(d), d, w.bqkv + 2 * d);
      put_v(src(d), d, w.bo);
      put_v(src(d), d, w.ln2g);
      put_v(src(d), d, w.ln2b);
      // cross attention: Q here, K/V into the fused all-layer cross-KV matrix
      put_t(src((int64_t)d * d), d, d, w.wqc);
      put_t(src((int64_t)d * d), d, d, wxkv + (size_t)(2 * i) * d * d);
      put_t(src((int64_t)d * d), d, d, wxkv + (size_t)(2 * i + 1) * d * d);
      put_t(src((int64_t)d * d), d, d, w.woc);
      put_v(src(d), d, w.bqc);
      put_v(src(d), d, bxkv + (size_t)2 * i * d);
      put_v(src(d), d, bxkv + (size_t)(2 * i + 1) * d);
      put_v(src(d), d, w.boc);
      put_v(src(d), d, w.ln3g);
      put_v(src(d), d, w.ln3b);
      put_t(src((int64_t)d * ff), d, ff, w.w1);
      put_v(src(ff), ff, w.b1);
      put_t(src((int64_t)ff * d), ff, d, w.w2);
      put_v(src(d), d, w.b2);
    }
    dec_lng = tvec(d);
    dec_lnb = tvec(d);
    put_v(src(d), d, dec_lng);
    put_v(src(d), d, dec_lnb);
    if (off != n) throw HrtError(HRT_ERR_INVALID, "parameter blob layout mismatch");
    // positional table (model.py:104-112): angles in fp64, cast to fp32
    std::vector<float> h_pe((size_t)P * d, 0.f);
    for (int p = 0; p < P; ++p)
      for (int i = 0; i < d / 2; ++i) {
        double ang = (double)p / std::pow(10000.0, 2.0 * i / d);
        h_pe[(size_t)p * d + 2 * i] = (float)std::sin(ang);
        h_pe[(size_t)p * d + 2 * i + 1] = (float)std::cos(ang);
      }
    pe = tvec((size_t)P * d);
    CUDA_OK(cudaMemcpyAsync(pe, h_pe.data(), h_pe.size() * sizeof(float), cudaMemcpyHostToDevice, stream));
    CUDA_OK(cudaStreamSynchronize(stream));
    cudaFree(dsrc);
    if (wp_hot != reinterpret_cast<T*>(wblob) + hot_bytes / sizeof(T))
      throw HrtError(HRT_ERR_INVALID, "hot weight region layout mismatch");
    set_l2_persist(l2_persist_mode);
    if constexpr (BF16) build_frag_weights();
  }

  // Fragment-native copies of every matrix the GEMV kernels read (gemv_small.cuh:
  // gv_frag_layout_kernel); the tcgen05 path keeps the K-major originals.
  char* fblob = nullptr;
  std::map<const void*, const T*> frag_map;
  void build_frag_weights() {
    std::vector<std::tuple<const T*, int, int>> mats;
    mats.emplace_back(E, V, d);
    for (const EncW& w : enc) {
      mats.emplace_back(w.wqkv, 3 * d, d);
      mats.emplace_back(w.wo, d, d);
      mats.emplace_back(w.w1, ff, d);
      mats.emplace_back(w.w2, d, ff);
    }
    mats.emplace_back(wxkv, Ld * 2 * d, d);
    for (const DecW& w : dec) {
      mats.emplace_back(w.wqkv, 3 * d, d);
      mats.emplace_back(w.wo, d, d);
      mats.emplace_back(w.wqc, d, d);
      mats.emplace_back(w.woc, d, d);
      mats.emplace_back(w.w1, ff, d);
      mats.emplace_back(w.w2, d, ff);
    }
    size_t total = 0;
    for (auto& m : mats)
      if (std::get<2>(m) % 32 == 0) total += gv_frag_elems(std::get<1>(m), std::get<2>(m));
    if (total == 0) return;
    CUDA_OK(cudaMalloc(&fblob, total * sizeof(T)));
    stats.weight_bytes += (int64_t)(total * sizeof(T));
    T* dst = reinterpret_cast<T*>(fblob);
    for (auto& m : mats) {
      const int N = std::get<1>(m), K = std::get<2>(m);
      if (K % 32) continue;  // the GEMV path requires K % 32 == 0
      const size_t n16 = gv_frag_elems(N, K) / 8;
      const int blocks = (int)std::min<size_t>((n16 + 255) / 256, 4096);
      gv_frag_layout_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const bf16*>(std::get<0>(m)), N, K,
                                                        reinterpret_cast<bf16*>(dst));
      check_launch();
      frag_map[std::get<0>(m)] = dst;
      dst += gv_frag_elems(N, K);
    }
    CUDA_OK(cudaStreamSynchronize(stream));
  }
  const T* frag_of(const T* W) const {
    auto it = frag_map.find(W);
    if (it == frag_map.end()) throw HrtError(HRT_ERR_INVALID, "GEMV weight without a fragment-native copy");
    return it->second;
  }

  // L2 persisting window over the Stage-I weights (launches on this stream,
  // captured graphs included): E and the decoder layers stay L2-resident while
  // the per-step K/V streams pass through
  size_t hot_bytes = 0;
  int l2_persist_mode = 0;  // option "l2_persist" (measured no effect at C2: off, leaves the device L2 limit alone)
  void set_l2_persist(int on) {
    l2_persist_mode = on;
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
    cudaStreamAttrValue av = {};
    if (on && max_persist > 0 && max_window > 0) {
      const size_t win = std::min(hot_bytes, (size_t)max_window);
      const size_t carve = std::min(win, (size_t)max_persist);
      CUDA_OK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
      av.accessPolicyWindow.base_ptr = wblob;
      av.accessPolicyWindow.num_bytes = win;
      av.accessPolicyWindow.hitRatio = std::min(1.0f, (float)carve / (float)win);
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      l2_window_bytes = win;
    } else {
      av.accessPolicyWindow.num_bytes = 0;
      l2_window_bytes = 0;
    }
    CUDA_OK(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &av));
  }
  size_t l2_window_bytes = 0;

  static int64_t param_count(const hrt_config& c) {
    int64_t d = c.d_model, f = c.d_ff;
    int64_t attn = 4 * d * d + 4 * d, ln = 2 * d, ffn = 2 * d * f + f + d;
    return (int64_t)c.vocab_size * d + c.enc_layers * (2 * ln + attn + ffn) + ln +
           c.dec_layers * (3 * ln + 2 * attn + ffn) + ln;
  }

  void transpose_convert(const float* s, int K, int N, T* dst);
  void convert(const float* s, size_t n, T* dst);

  // -------------------------------------------------------------------------
  // capacity + arena plan
  // -------------------------------------------------------------------------
  // Arena dimensions: the engine's capacity (max_dims), or one call's actual
  // sizes when accounting the high-water mark. One closed form serves the
  // allocation, the high-water mark and hrt_estimate_arena (estimate_max_bytes,
  // infer.py:78-96).
  struct ArenaDims {
    int Me, R, M2, Mm;
  };
  static ArenaDims max_dims(const hrt_config& c) {
    const int B = std::max(1, c.max_sentences), beam = std::max(1, c.max_beam);
    const int M2 = B * beam * (c.max_len + c.max_chunk);
    return ArenaDims{c.max_src_tokens > 0 ? c.max_src_tokens : B * c.max_len, B * beam, M2, M2};
  }
  void size_capacity() {
    const ArenaDims a = max_dims(cfg);
    Bmax = std::max(1, cfg.max_sentences);
    beam_max = std::max(1, cfg.max_beam);
    Me_max = a.Me;
    R_max = a.R;
    cap_max = Lmax + 1;  // AT mode (k = 1) worst case; skip-AT needs ceil(L/k)+1
    M2_max = a.M2;
    Mm_max = a.Mm;
    nt_max = cdiv(V, 64);
    logit_rows = 4096;
  }
  // largest phase footprint of a call with these sizes (arena_high_water)
  void note_high_water(int phase, const ArenaDims& a) {
    Plan p;
    carve_plan(phase, p, nullptr, a, cfg, nullptr);
    stats.arena_high_water = std::max<int64_t>(stats.arena_high_water, (int64_t)p.off);
  }

  template <class Fn>
  size_t plan_phases(char* base, Fn&& assign) {
    size_t mx = 0;
    for (int phase = 0; phase < 3; ++phase) {
      Plan p;
      assign(phase, p, base);
      mx = std::max(mx, p.off);
    }
    return mx;
  }

  // vocab GEMM tile width: 256 whenever the vocabulary is large (fewer
  // partials per row for the selection merge, one tile per CTA at small R)
  int vocab_bn(int rows) const { return V >= 4096 ? 256 : std::max(64, choose_bn(rows, V)); }  // row-wise epilogue: column halves
  // upper bound on vocab tiles per row for any row count (partials sizing)
  static int nt_bound(const hrt_config& c) {
    return (BF16 && c.vocab_size < 4096) ? cdiv(c.vocab_size, 32) : cdiv(c.vocab_size, 128);
  }
  static void estimate(const hrt_config& c, int64_t* phase_bytes) {
    const ArenaDims a = max_dims(c);
    int64_t mx = 0;
    for (int ph = 0; ph < 3; ++ph) {
      Plan p;
      carve_plan(ph, p, nullptr, a, c, nullptr);
      phase_bytes[ph] = (int64_t)p.off;
      mx = std::max(mx, phase_bytes[ph]);
    }
    phase_bytes[3] = mx;
  }

  static void carve_plan(int phase, Plan& p, char* base, const ArenaDims& a, const hrt_config& c, Engine* e) {
    const int d = c.d_model, ff = c.d_ff, Ld = c.dec_layers, V = c.vocab_size, cap_max = c.max_len + 1;
    const int logit_rows = 4096;
    const int Me_max = a.Me, R_max = a.R, M2_max = a.M2, Mm_max = a.Mm;
    EncBufs eb_{};
    S1Bufs s1_{};
    S2Bufs s2_{};
    EncBufs& eb = e ? e->eb : eb_;
    S1Bufs& s1 = e ? e->s1 : s1_;
    S2Bufs& s2 = e ? e->s2 : s2_;
    if (phase == 0) {
      eb.x = p.take<float>(base, (size_t)Me_max * d);
      eb.y = p.take<T>(base, (size_t)Me_max * d);
      eb.qkv = p.take<T>(base, (size_t)Me_max * 3 * d);
      eb.ctx = p.take<T>(base, (size_t)Me_max * d);
      eb.hid = p.take<T>(base, (size_t)Me_max * ff);
    } else if (phase == 1) {
      s1.x = p.take<float>(base, (size_t)R_max * d);
      s1.y = p.take<T>(base, (size_t)R_max * d);
      s1.qkv = p.take<T>(base, (size_t)R_max * 3 * d);
      s1.qc = p.take<T>(base, (size_t)R_max * d);
      s1.ctx = p.take<T>(base, (size_t)R_max * d);
      s1.hid = p.take<T>(base, (size_t)R_max * ff);
      s1.kc = p.take<T>(base, (size_t)Ld * R_max * cap_max * d);
      s1.vc = p.take<T>(base, (size_t)Ld * R_max * cap_max * d);
      const size_t ntot = (size_t)R_max * nt_bound(c);
      s1.parts.mx = p.take<float>(base, ntot);
      s1.parts.sum = p.take<float>(base, ntot);
      s1.parts.val = p.take<float>(base, ntot * KTOP_MAX);
      s1.parts.id = p.take<int>(base, ntot * KTOP_MAX);
      s1.parts.eos = p.take<float>(base, R_max);
      s1.rowstat = p.take<RowStat>(base, R_max);
      s1.logits = p.take<float>(base, (size_t)std::min(R_max, logit_rows) * V);
    } else {
      s2.x = p.take<float>(base, (size_t)M2_max * d);
      s2.y = p.take<T>(base, (size_t)M2_max * d);
      s2.qkv = p.take<T>(base, (size_t)M2_max * 3 * d);
      s2.qc = p.take<T>(base, (size_t)M2_max * d);
      s2.ctx = p.take<T>(base, (size_t)M2_max * d);
      s2.hid = p.take<T>(base, (size_t)M2_max * ff);
      s2.ymask = p.take<T>(base, (size_t)Mm_max * d);
      s2.ids = p.take<int>(base, M2_max);
      s2.pos = p.take<int>(base, M2_max);
      s2.out_row = p.take<int>(base, M2_max);
      const size_t ntot = (size_t)Mm_max * nt_bound(c);
      s2.parts.mx = p.take<float>(base, ntot);
      s2.parts.sum = p.take<float>(base, ntot);
      s2.parts.val = p.take<float>(base, ntot);  // KT = 1 in Stage II
      s2.parts.id = p.take<int>(base, ntot);
      s2.parts.eos = p.take<float>(base, Mm_max);
      s2.mstat = p.take<RowStat>(base, Mm_max);
      s2.logits = p.take<float>(base, (size_t)std::min(Mm_max, logit_rows) * V);
    }
  }

  void alloc_buffers() {
    // persistent region
    meta_cap = 16 * Bmax * beam_max + 10 * M2_max + 2 * V + 256 + 8 + 2 * (cap_max + 8) + 2 * (R_max + 16) +
               Me_max + Bmax + 8;  // + the call's source ids
    auto persist_plan = [&](char* base) {
      Plan p;
      d_ids_raw = p.take<int>(base, Me_max + Bmax);
      d_ids = p.take<int>(base, Me_max);
      d_pos = p.take<int>(base, Me_max);
      d_meta = p.take<int>(base, meta_cap);
      xkv = p.take<T>(base, (size_t)Me_max * Ld * 2 * d);
      s_feed = p.take<int>(base, R_max);
      s_done = p.take<int>(base, R_max);
      s_nsteps = p.take<int>(base, R_max);
      s_forced = p.take<int>(base, R_max);
      s_caps = p.take<int>(base, R_max);
      s_rowseq = p.take<int>(base, R_max);
      s_parents = p.take<int>(base, R_max);
      s_anchors = p.take<int>(base, (size_t)R_max * cap_max);
      s_hist = p.take<int>(base, (size_t)R_max * cap_max);
      s_hist2 = p.take<int>(base, (size_t)R_max * cap_max);
      s_score = p.take<double>(base, R_max);
      b_greedy = p.take<int>(base, R_max);
      b_anchors2 = p.take<int>(base, (size_t)R_max * cap_max);
      b_live = p.take<int>(base, Bmax);
      b_nfin = p.take<int>(base, Bmax);
      b_gdone = p.take<int>(base, Bmax);
      b_fcount = p.take<int>(base, Bmax);
      b_fgslot = p.take<int>(base, Bmax);
      b_flist = p.take<int>(base, (size_t)Bmax * beam_max);
      b_fscore = p.take<double>(base, (size_t)Bmax * (beam_max + 2));
      b_flen = p.take<int>(base, (size_t)Bmax * (beam_max + 2));
      b_fforced = p.take<int>(base, (size_t)Bmax * (beam_max + 2));
      b_ftok = p.take<int>(base, (size_t)Bmax * (beam_max + 2) * cap_max);
      c_off = p.take<int>(base, (size_t)Bmax * beam_max);
      c_len = p.take<int>(base, (size_t)Bmax * beam_max);
      c_sat = p.take<double>(base, (size_t)Bmax * beam_max);
      c_forced = p.take<int>(base, (size_t)Bmax * beam_max);
      o_tokens = p.take<int>(base, (size_t)Bmax * Lmax);
      o_lens = p.take<int>(base, Bmax);
      o_calls = p.take<int>(base, Bmax);
      o_scores = p.take<double>(base, (size_t)Bmax * 3);
      o_forced = p.take<unsigned char>(base, Bmax);
      return p.off;
    };
    size_t pbytes = persist_plan(nullptr);
    CUDA_OK(cudaMalloc(&persist, pbytes));
    persist_plan(persist);
    CUDA_OK(cudaMemset(persist, 0, pbytes));
    // fixed header of the metadata buffer: Stage-I loop control, alive[],
    // source offsets / lengths (graph-captured kernels keep these pointers)
    // source offsets / lengths are sized for R_max rows: graph launches cover a
    // power-of-two row bucket, and rows past the live sentences read length 0
    meta_hdr = 8 + align_up(cap_max + 1, 8) + align_up(R_max + 1, 8) + align_up(R_max, 8);
    s_ctl = reinterpret_cast<StepCtl*>(d_meta);
    s_alive = d_meta + 8;
    s_srcoff = s_alive + align_up(cap_max + 1, 8);
    s_srclen = s_srcoff + align_up(R_max + 1, 8);
    arena_bytes = 0;
    const ArenaDims amax = max_dims(cfg);
    for (int ph = 0; ph < 3; ++ph) {
      Plan p;
      carve_plan(ph, p, nullptr, amax, cfg, this);
      arena_bytes = std::max(arena_bytes, p.off);
    }
    cudaError_t e = cudaMalloc(&arena, arena_bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw HrtError(HRT_ERR_MEMORY, "device arena of " + std::to_string(arena_bytes) + " bytes: " +
                                         cudaGetErrorString(e));
    }
    for (int ph = 0; ph < 3; ++ph) {
      Plan p;
      carve_plan(ph, p, arena, amax, cfg, this);
    }
    // the activation arena (phases alias); the persistent handoff region (cross-K/V,
    // Stage-I state, I/O staging) lives outside it, like the reference session's
    // memory / cross_k / cross_v (infer.py:156-160)
    stats.arena_bytes = (int64_t)arena_bytes;
    if (BF16) {
      CUDA_OK(cudaMalloc(&sk_ws, sk_ws_bytes));
      CUDA_OK(cudaMalloc(&sk_counters, sk_max_tiles * sizeof(int)));
      CUDA_OK(cudaMemset(sk_counters, 0, sk_max_tiles * sizeof(int)));
      CUDA_OK(cudaMalloc(&gv_counter, 64 * sizeof(int)));
      CUDA_OK(cudaMemset(gv_counter, 0, 64 * sizeof(int)));
    }
    CUDA_OK(cudaMallocHost(&h_meta, (size_t)meta_cap * sizeof(int)));
    CUDA_OK(cudaMallocHost(&h_ctl, sizeof(StepCtl)));
    h_out_bytes = (size_t)Bmax * Lmax * sizeof(int) + 2 * (size_t)Bmax * sizeof(int) + 8 + (size_t)Bmax * 3 * sizeof(double) + Bmax;
    CUDA_OK(cudaMallocHost(&h_out, h_out_bytes));
    CUDA_OK(cudaEventCreateWithFlags(&meta_ev, cudaEventDisableTiming));
    CUDA_OK(cudaEventRecord(meta_ev, stream));
  }

  // -------------------------------------------------------------------------
  // kernel launch wrappers
  // -------------------------------------------------------------------------
  const CUtensorMap& tmap(const void* p, int rows, int cols, int ld, int box) {
    auto key = std::make_tuple(p, rows, cols, ld, box);
    auto it = tmaps.find(key);
    if (it != tmaps.end()) return it->second;
    return tmaps.emplace(key, make_tmap_bf16_kmajor(p, rows, cols, ld, box)).first->second;
  }

  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> tmaps_out;
  template <class Epi>
  const CUtensorMap& tmap_out(const Epi& epi, int rows, int cols, const CUtensorMap& dummy) {
    if constexpr (EpiTmaStore<Epi>::value) {
      auto key = std::make_tuple(static_cast<const void*>(epi.out), rows, cols, epi.ldo);
      auto it = tmaps_out.find(key);
      if (it != tmaps_out.end()) return it->second;
      return tmaps_out.emplace(key, make_tmap_bf16_store(epi.out, rows, cols, epi.ldo)).first->second;
    } else {
      (void)epi;
      (void)rows;
      (void)cols;
      return dummy;
    }
  }
  // split-K workspace: fp32 partial tiles + per-tile arrival counters
  float* sk_ws = nullptr;
  int* sk_counters = nullptr;
  size_t sk_ws_bytes = (size_t)64 << 20;
  int sk_max_tiles = 16384;
  int* gv_counter = nullptr;  // GEMV LayerNorm-tail arrival counter
  bool use_splitk = false;  // measured slower than unsplit on B200 (fix-up tail); option "splitk"
  int choose_splits(int M, int N, int K, int bn) const {
    if (!use_splitk) return 1;
    const int tiles = cdiv(N, bn) * cdiv(M, TC_BM);
    const int kb = K / TC_BK;
    int S = 1;
    while (S * 2 <= 8 && tiles * S * 2 <= num_sms && kb / (S * 2) >= 2) S *= 2;
    while (S > 1 && (size_t)S * cdiv(M, TC_BM) * TC_BM * N * sizeof(float) > sk_ws_bytes) S /= 2;
    if (tiles > sk_max_tiles) S = 1;
    return S;
  }

  template <int BN, int ST, class Epi, int CL, bool PAIR = false>
  void tc_launch_cl(const T* A, int a_cap, int lda, int M, const T* W, int N, int K, const Epi& epi,
                    const int* M_dev) {
    if constexpr (BF16) {
      auto kern = tc_gemm_kernel<BN, ST, Epi, CL, PAIR>;
      const int smem = TcSmem<BN, ST, PAIR ? BN / 2 : BN>::TOTAL;
      smem_optin(kern, smem);
      const CUtensorMap& ta = tmap(A, a_cap, K, lda, TC_BM);
      const CUtensorMap& tb = tmap(W, N, K, K, BN / CL);
      // bf16 element-wise outputs leave through TMA tile stores (the buffer holds a_cap rows)
      const CUtensorMap& tc = tmap_out<Epi>(epi, a_cap, N, ta);
      SplitK sk{1, sk_ws, sk_counters};
      if constexpr (!Epi::kRowWise && CL == 1) sk.splits = choose_splits(M, N, K, BN);
      if constexpr (std::is_same<Epi, EpiResidual>::value) {
        if (res_red && sk.splits == 1) {
          Epi e2 = epi;
          e2.red = true;
          const int units = cdiv(N, BN) * cdiv(cdiv(M, TC_BM), CL);
          const int grid = grid_clusters(units, resident_clusters(kern, smem, CL)) * CL;
          launch_cluster = CL;
          launch(kern, grid, TC_THREADS, smem, ta, tb, tc, M, N, K, M_dev, e2, sk);
          launch_cluster = 1;
          return;
        }
      }
      // M: count, or upper bound with M_dev; CL = 2 works on vertical tile pairs
      const int units = cdiv(N, BN) * cdiv(cdiv(M, TC_BM), CL) * sk.splits;
      const int grid = grid_clusters(units, resident_clusters(kern, smem, CL)) * CL;
      launch_cluster = CL;
      launch(kern, grid, TC_THREADS, smem, ta, tb, tc, M, N, K, M_dev, epi, sk);
      launch_cluster = 1;
    }
  }
  // Clusters of CL CTAs (one per SM) that can be resident at once: a persistent grid
  // larger than that would run its last clusters as a second wave. GPCs hold
  // different SM counts, so this can be below num_sms / CL.
  std::map<std::pair<const void*, int>, int> resident_cache;
  // option "sm_cap": SMs a persistent tcgen05 grid may occupy (0 = all). Below the SM count,
  // the remaining SMs stay free for the latency-bound Stage-I kernels of other engines
  // (pipelined batches on other streams) while this engine's large GEMMs run.
  int sm_cap = 0;
  // option "balance": a persistent grid of as many clusters as the rounds need (same
  // number of rounds as the full grid, fewer idle SMs in the last one: they stay free
  // for the other engines' kernels when batches pipeline)
  bool balance = true;
  int grid_clusters(int units, int maxc) const {
    if (!balance || units <= maxc) return std::min(units, maxc);
    const int rounds = cdiv(units, maxc);
    return cdiv(units, rounds);
  }
  template <class K>
  int resident_clusters(K kern, int smem, int CL) {
    const int cap = sm_cap > 0 ? std::max(1, std::min(num_sms, sm_cap) / CL) : num_sms;
    return std::min(cap, resident_clusters_all(kern, smem, CL));
  }
  template <class K>
  int resident_clusters_all(K kern, int smem, int CL) {
    if (CL == 1) return num_sms;
    auto key = std::make_pair(reinterpret_cast<const void*>(kern), CL);
    auto it = resident_cache.find(key);
    if (it != resident_cache.end()) return it->second;
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(CL * (num_sms / CL));
    c.blockDim = dim3(TC_THREADS);
    c.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    c.attrs = at;
    c.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &c) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms / CL;
    }
    n = std::min(n, num_sms / CL);
    resident_cache[key] = n;
    if (getenv("HRT_DEBUG_CLUSTERS")) fprintf(stderr, "resident clusters of %d: %d\n", CL, n);
    return n;
  }
  // CTA pairs sharing the weight tile (multicast) once there are enough row
  // tiles to pair up (large-batch encoder / Stage II / vocabulary GEMMs)
  int cluster_mode = 1;  // option "cluster"
  int cluster_min_mtiles = 16;
  // clusters of four CTAs sharing the weight tile (a quarter each, multicast): option
  // "cluster4" (1 = on), from cluster4_min_mtiles row tiles up (8 for the vocabulary)
  int cluster4 = 0;
  int cluster4_min_mtiles = 32;
  template <int BN, int ST, class Epi>
  void tc_launch(const T* A, int a_cap, int lda, int M, const T* W, int N, int K, const Epi& epi, const int* M_dev) {
    const int mt = cdiv(M, TC_BM);
    // wide-N GEMMs (vocabulary) pair up from 4 row tiles: their weight stream dominates L2 -> SM traffic
    if (cluster4 && !pair_mma && (mt >= cluster4_min_mtiles || (mt >= 8 && N >= 8192)) &&
        choose_splits(M, N, K, BN) == 1) {
      tc_launch_cl<BN, ST, Epi, 4>(A, a_cap, lda, M, W, N, K, epi, M_dev);
      return;
    }
    if (cluster_mode && (mt >= cluster_min_mtiles || (mt >= 4 && N >= 8192)) && choose_splits(M, N, K, BN) == 1) {
      // cta_group::2 pairs (option "pair"): half the weight tile per CTA, so more ring stages
      if constexpr (BN >= 128) {
        if (pair_mma) {
          tc_launch_cl<BN, BN == 256 ? 6 : 8, Epi, 2, true>(A, a_cap, lda, M, W, N, K, epi, M_dev);
          return;
        }
      }
      tc_launch_cl<BN, ST, Epi, 2>(A, a_cap, lda, M, W, N, K, epi, M_dev);
    }
    else
      tc_launch_cl<BN, ST, Epi, 1>(A, a_cap, lda, M, W, N, K, epi, M_dev);
  }

  // widest N tile that still fills ~0.6 of the SMs (large-M encoder / Stage-II
  // GEMMs -> 256, Stage-I GEMMs with few row tiles -> 128 or 64)
  int pair_mma = 0;  // option "pair": CTA-pair GEMMs as cta_group::2 MMAs instead of multicast weight tiles
  int bn32_mode = 1;  // option "bn32": 32-column tiles when 64-column tiles leave most SMs idle
  int fill_pct = 60;  // option "fill": SM share the widest tile must still reach
  int choose_bn(int M, int N) const {
    const int mt = cdiv(M, TC_BM);
    if (M > 128)
      for (int bn : {256, 128})
        if (mt * cdiv(N, bn) * 100 >= num_sms * fill_pct) return bn;
    if (bn32_mode && mt * cdiv(N, 64) * 2 < num_sms) return 32;
    return 64;
  }

  // small-M regime (decode steps at small batch, batch-1 encoder / Stage II):
  // mma.sync GEMV with K split over the warps of a CTA (gemv_small.cuh)
  bool use_gemv = true;  // option "gemv"
  int gemv_max_m = 64;  // option "gemv_max_m" (32, 64 or 128; measured best: 64)
  // path_rows: when set (eager Stage-I loop), the kernel choice follows the
  // captured graph's row bucket instead of the live row count, so eager and
  // graph launches run the same kernels (bit-identical results)
  int path_rows = 0;
  // fp32 GEMV route (gemv_f32_kernel) for up to gemv_f32_max_m rows; false when the shape does not fit
  static constexpr int gemv_f32_max_m = 32;
  template <class Epi>
  bool gemv_f32(const T* A, int lda, const T* W, int N, int K, int M, int Mp, const int* M_dev, const Epi& epi) {
    // up to 32 rows always; up to 256 while the 64x64-tile SIMT grid would leave SMs idle
    const bool small = Mp <= gemv_f32_max_m || (Mp <= 256 && cdiv(Mp, SG_BM) * cdiv(N, SG_BN) < num_sms);
    if (BF16 || !use_gemv || !small || K % 128 != 0 || K > 16 * 128 || lda % 4 != 0) return false;
    const float* Af = reinterpret_cast<const float*>(A);
    const float* Wf = reinterpret_cast<const float*>(W);
    const dim3 grid(cdiv(N, GF_WARPS), cdiv(Mp, GF_MAXM));
    switch (K / 128) {
      case 1: launch(gemv_f32_kernel<1, Epi>, grid, GF_WARPS * 32, 0, Af, lda, Wf, N, K, M, M_dev, epi); break;
      case 2: launch(gemv_f32_kernel<2, Epi>, grid, GF_WARPS * 32, 0, Af, lda, Wf, N, K, M, M_dev, epi); break;
      case 4: launch(gemv_f32_kernel<4, Epi>, grid, GF_WARPS * 32, 0, Af, lda, Wf, N, K, M, M_dev, epi); break;
      case 8: launch(gemv_f32_kernel<8, Epi>, grid, GF_WARPS * 32, 0, Af, lda, Wf, N, K, M, M_dev, epi); break;
      case 16: launch(gemv_f32_kernel<16, Epi>, grid, GF_WARPS * 32, 0, Af, lda, Wf, N, K, M, M_dev, epi); break;
      default: return false;
    }
    return true;
  }
  // row-blocked GEMV (blockIdx.y = 64-row blocks) up to gemv_rows rows: at these row counts
  // the tcgen05 tile pipeline is pure fixed latency (option "gemv_rows", 0 = off)
  int gemv_rows = 128;  // measured: R = 128 step 71.4 -> 61.2 us; no gain at 256, slower at 512
  bool gemv_ok(int M, int K) const {
    const int Mp = path_rows > 0 ? path_rows : M;
    return use_gemv && Mp <= std::max(gemv_max_m, gemv_rows) && K % 32 == 0 &&
           (K <= 512 || (K / 32) % GV_WARPS == 0) && K <= 4096;
  }
  // the vocabulary GEMV keeps per-row statistics in registers: at most 32 rows
  bool gemv_vocab_ok(int M) const {
    const int Mp = path_rows > 0 ? path_rows : M;
    return gemv_ok(M, d) && Mp <= 32;
  }
  template <int NT, int CPW, bool LNA, bool TLN, class Epi>
  void gemv_launch_t(const T* A, int lda, int M, const T* W, int N, int K, const Epi& epi, const int* M_dev,
                     const GvLN& ln, const GvTailLN& tln) {
    const int ry = cdiv(M, 8 * NT);  // 64-row blocks beyond 64 rows (NT = 8)
    if (ry > 1 && (LNA || TLN)) throw HrtError(HRT_ERR_INVALID, "GEMV LayerNorm fusion needs <= 64 rows");
    launch(gemv_small_kernel<NT, CPW, Epi, LNA, TLN>, dim3(cdiv(N, 16), ry), GV_THREADS, 0,
           reinterpret_cast<const bf16*>(A), lda, reinterpret_cast<const bf16*>(frag_of(W)), N, K, M, M_dev, epi, ln,
           tln);
  }
  template <int NT, bool LNA, bool TLN, class Epi>
  void gemv_launch_n(const T* A, int lda, int M, const T* W, int N, int K, const Epi& epi, const int* M_dev,
                     const GvLN& ln, const GvTailLN& tln) {
    const int cpw = std::max(1, K / 32 / GV_WARPS);
    if (cpw == 1) gemv_launch_t<NT, 1, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else if (cpw == 2) gemv_launch_t<NT, 2, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else if (cpw == 4) gemv_launch_t<NT, 4, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else gemv_launch_t<NT, 8, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
  }
  template <bool LNA = false, bool TLN = false, class Epi>
  void gemv_launch(const T* A, int lda, int M, const T* W, int N, int K, const Epi& epi, const int* M_dev,
                   const GvLN& ln = GvLN{nullptr, nullptr, nullptr},
                   const GvTailLN& tln = GvTailLN{nullptr, nullptr, nullptr, nullptr}) {
    if (M <= 8) gemv_launch_n<1, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else if (M <= 16) gemv_launch_n<2, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else if (M <= 32) gemv_launch_n<4, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else if (M <= 64 || gemv_max_m <= 64) gemv_launch_n<8, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
    else gemv_launch_n<16, LNA, TLN>(A, lda, M, W, N, K, epi, M_dev, ln, tln);
  }
  // residual projection followed by a LayerNorm of the updated rows: on the
  // GEMV path the last CTA normalises (no LN launch), else GEMM + LN kernel
  bool use_tail_ln = false;  // option "tail_ln" (measured slower than the separate LN launch: off)
  bool tail_ln_ok(int M, int K) const {
    const int Mp = path_rows > 0 ? path_rows : M;
    return BF16 && use_tail_ln && Mp <= 64 && gemv_ok(M, K) && d % 128 == 0 && d <= 1024;
  }
  // residual + LayerNorm in the tcgen05 epilogue (tc_gemm_ln.cuh): rows above the GEMV
  // regime, d a multiple of 256 with d / 256 in {1, 2, 4} (a cluster of d / 256 CTAs per row block)
  // residual GEMM epilogues (tcgen05, no split-K) as L2 reductions: option "res_red"
  bool res_red = true;
  bool use_ln_epi = false;  // option "ln_epi" (correct, measured slower than GEMM + LN kernel: off)
  bool ln_epi_ok(int M, int K) const {
    const int nc = d / TL_BN;
    return BF16 && use_ln_epi && !gemv_ok(M, K) && d % TL_BN == 0 && (nc == 1 || nc == 2 || nc == 4) &&
           K % TC_BK == 0;
  }
  // full-row form (tc_gemm_lnrow.cuh, d = 512): option "ln_row" = 1 TMA-staged lane-per-row
  // epilogue with the updated rows kept in TMEM, 2 / 3 register epilogue re-reading them from
  // L2 (accumulator released after pass 1) / keeping them in TMEM; used
  // from ln_row_min_tiles 128-row blocks up (Stage-I buckets keep the narrow-tile GEMM + LN)
  int ln_row = 1;
  int ln_row_min_tiles = 16;
  bool ln_row_ok(int M, int K) const {
    return BF16 && ln_row != 0 && d == LR_D && K % TC_BK == 0 && cdiv(M, TC_BM) >= ln_row_min_tiles &&
           !gemv_ok(M, K);
  }
  std::map<std::tuple<const void*, int>, CUtensorMap> tmaps_x;
  template <int MODE, int ST = 3>
  void lnrow_launch(const T* A, int a_cap, int lda, int M, const T* W, int K, const ResLnArgs& ra,
                    const int* M_dev) {
    if constexpr (BF16) {
      // ST x 48 KB operand ring (+ 32 KB per-warp buffers unless MODE 2 borrows 4 stages) + statistics
      auto kern = tc_gemm_resln_row_kernel<ST, MODE>;
      const int smem = LrSmem<ST, lr_stg<ST, MODE>()>::TOTAL;
      smem_optin(kern, smem);
      const CUtensorMap& ta = tmap(A, a_cap, K, lda, TC_BM);
      const CUtensorMap& tb = tmap(W, d, K, K, LR_D / 4);
      auto key = std::make_tuple(static_cast<const void*>(ra.x), M);
      auto itx = tmaps_x.find(key);
      if (itx == tmaps_x.end()) itx = tmaps_x.emplace(key, make_tmap_f32_tile(ra.x, M, d, ra.ldx)).first;
      const int grid = grid_clusters(cdiv(cdiv(M, TC_BM), 2), resident_clusters(kern, smem, 2)) * 2;
      launch_cluster = 2;
      launch(kern, grid, TC_THREADS, smem, ta, tb, itx->second, M, K, M_dev, ra);
      launch_cluster = 1;
    }
  }
  template <int NC>
  void resln_launch(const T* A, int a_cap, int lda, int M, const T* W, int K, const ResLnArgs& ra,
                    const int* M_dev) {
    if constexpr (BF16) {
      constexpr int ST = 3;  // 3 x 48 KB ring + 32 KB transpose buffers + row statistics
      auto kern = tc_gemm_resln_kernel<NC, ST>;
      const int smem = TlSmem<NC, ST>::TOTAL;
      smem_optin(kern, smem);
      const CUtensorMap& ta = tmap(A, a_cap, K, lda, TC_BM);
      const CUtensorMap& tb = tmap(W, d, K, K, TL_BN);
      const int grid = std::min(cdiv(M, TC_BM), resident_clusters(kern, smem, NC)) * NC;
      launch_cluster = NC;
      launch(kern, grid, TC_THREADS, smem, ta, tb, M, K, M_dev, ra);
      launch_cluster = 1;
    }
  }
  // x += A W^T + bias, then y = LN(x) (rows out_row[r] of y when given): one fused
  // launch on the tcgen05 path, GEMV tail-LN or GEMM + LN kernel otherwise
  // "<current tag><suffix>" (timing attribution of a call site's trailing launch)
  std::map<std::pair<const char*, const char*>, std::string> sub_tags;
  const char* sub_tag(const char* suffix) {
    if (cur_tag == nullptr) return nullptr;
    std::string& t = sub_tags[{cur_tag, suffix}];
    if (t.empty()) t = std::string(cur_tag) + suffix;
    return t.c_str();
  }
  void gemm_res_ln(const T* A, int a_cap, int lda, int M, const T* W, int K, float* x, const float* bias,
                   const float* g, const float* b, T* y, const int* M_dev, const int* out_row = nullptr) {
    if (M <= 0) return;
    if (ln_row_ok(M, K)) {
      Scope sc(this, K_GEMM, (double)sizeof(T) * ((double)d * K + (double)M * K), 2.0 * M * d * K);
      const ResLnArgs ra{x, d, bias, g, b, reinterpret_cast<bf16*>(y), d, out_row};
      if (ln_row == 2) lnrow_launch<0>(A, a_cap, lda, M, W, K, ra, M_dev);
      else if (ln_row == 3) lnrow_launch<1>(A, a_cap, lda, M, W, K, ra, M_dev);
      else if (ln_row == 4) lnrow_launch<2, 4>(A, a_cap, lda, M, W, K, ra, M_dev);
      else lnrow_launch<2>(A, a_cap, lda, M, W, K, ra, M_dev);
      check_launch();
      return;
    }
    if (ln_epi_ok(M, K)) {
      Scope sc(this, K_GEMM, (double)sizeof(T) * ((double)d * K + (double)M * K), 2.0 * M * d * K);
      const ResLnArgs ra{x, d, bias, g, b, reinterpret_cast<bf16*>(y), d, out_row};
      const int nc = d / TL_BN;
      if (nc == 1) resln_launch<1>(A, a_cap, lda, M, W, K, ra, M_dev);
      else if (nc == 2) resln_launch<2>(A, a_cap, lda, M, W, K, ra, M_dev);
      else resln_launch<4>(A, a_cap, lda, M, W, K, ra, M_dev);
      check_launch();
      return;
    }
    if (tail_ln_ok(M, K)) {
      Scope sc(this, K_GEMM, (double)sizeof(T) * ((double)d * K + (double)M * K), 2.0 * M * d * K);
      gemv_launch<false, true>(A, lda, M, W, d, K, EpiResidual{x, d, bias}, M_dev, GvLN{nullptr, nullptr, nullptr},
                               GvTailLN{g, b, reinterpret_cast<bf16*>(y), gv_counter});
      check_launch();
      return;
    }
    gemm(K_GEMM, A, a_cap, lda, M, W, d, K, EpiResidual{x, d, bias}, M_dev);
    Tag _t(this, sub_tag(".ln"));
    layernorm(x, M, g, b, y, out_row, nullptr, M_dev);
  }
  // LayerNorm feeding a projection: fused into the GEMV prologue on the
  // small-M path (bit-identical operand), else LN kernel + GEMM
  bool use_ln_fuse = false;  // option "ln_fuse" (measured: no faster than LN kernel + GEMV at B = 1)
  bool ln_fusable(int M) const { return use_ln_fuse && BF16 && gemv_vocab_ok(M) && d % 128 == 0 && d <= 1024; }
  template <class Epi>
  void gemm_ln(int cls, const float* x, const float* g, const float* b, T* y, int y_cap, int M, const T* W, int N,
               const Epi& epi, const int* M_dev) {
    if (M <= 0) return;
    if (ln_fusable(M)) {
      Scope sc(this, cls, (double)sizeof(T) * N * d + 4.0 * M * d, 2.0 * M * N * d);
      gemv_launch<true>(y, d, M, W, N, d, epi, M_dev, GvLN{x, g, b});
      check_launch();
      return;
    }
    layernorm(x, M, g, b, y, nullptr, nullptr, M_dev);
    gemm(cls, y, y_cap, d, M, W, N, d, epi, M_dev);
  }

  // C[M,N] = A[M,K] . W[N,K]^T with a fused epilogue
  template <class Epi>
  void gemm(int cls, const T* A, int a_cap, int lda, int M, const T* W, int N, int K, const Epi& epi,
            const int* M_dev = nullptr, int bn = 0) {
    if (M <= 0) return;
    Scope sc(this, cls, (double)sizeof(T) * ((double)N * K + (double)M * K), 2.0 * M * N * K);
    if constexpr (BF16) {
      if (gemv_ok(M, K)) {
        gemv_launch(A, lda, M, W, N, K, epi, M_dev);
        check_launch();
        return;
      }
      if (bn == 0) bn = choose_bn(M, N);
      if (bn == 32)
        tc_launch<32, 8>(A, a_cap, lda, M, W, N, K, epi, M_dev);
      else if (bn == 64)
        tc_launch<64, 8>(A, a_cap, lda, M, W, N, K, epi, M_dev);
      else if (bn == 128)
        tc_launch<128, 6>(A, a_cap, lda, M, W, N, K, epi, M_dev);
      else
        tc_launch<256, 4>(A, a_cap, lda, M, W, N, K, epi, M_dev);
    } else {
      const int Mp = path_rows > 0 ? path_rows : M;
      if (!gemv_f32(A, lda, W, N, K, M, Mp, M_dev, epi)) {
        dim3 grid(cdiv(N, SG_BN), cdiv(M, SG_BM));
        launch(simt_gemm_kernel<T, Epi>, grid, SG_THREADS, 0, A, lda, W, K, M, N, K, M_dev, epi,
                                                                   epi.ld() % 4 == 0);
      }
    }
    check_launch();
  }

  template <int NPL>
  void ln_launch(const float* x, const int* M_dev, int M, const float* g, const float* b, T* y, const int* out_row,
                 float* y32) {
    launch(layernorm_kernel<T, NPL>, cdiv(M, 8), 256, 0, x, M_dev, M, d, g, b, y, out_row, y32);
  }
  void layernorm(const float* x, int M, const float* g, const float* b, T* y, const int* out_row = nullptr,
                 float* y32 = nullptr, const int* M_dev = nullptr) {
    if (M <= 0) return;
    Scope sc(this, K_OTHER, (double)M * d * (4 + sizeof(T)), 8.0 * M * d);
    if (d % 128 == 0 && d <= 1024) {
      const int nv = d / 128;
#define HRT_LNV(N) launch(layernorm_vec_kernel<T, N>, cdiv(M, 8), 256, 0, x, M_dev, M, d, g, b, y, out_row, y32)
      if (nv == 1) HRT_LNV(1);
      else if (nv == 2) HRT_LNV(2);
      else if (nv == 4) HRT_LNV(4);
      else if (nv == 8) HRT_LNV(8);
      else goto scalar_ln;
#undef HRT_LNV
      check_launch();
      return;
    }
  scalar_ln:
    const int npl = cdiv(d, 32);
#define HRT_LN(N) ln_launch<N>(x, M_dev, M, g, b, y, out_row, y32)
    if (npl <= 1) HRT_LN(1);
    else if (npl <= 2) HRT_LN(2);
    else if (npl <= 4) HRT_LN(4);
    else if (npl <= 8) HRT_LN(8);
    else if (npl <= 16) HRT_LN(16);
    else HRT_LN(32);
#undef HRT_LN
    check_launch();
  }

  template <int NPL>
  void emb_launch(const int* ids, const int* pos, int pc, const int* pos_dev, const int* M_dev, int M, const float* g,
                  const float* b, float* x, T* y) {
    launch(embed_ln_kernel<T, NPL>, cdiv(M, 8), 256, 0, ids, pos, pc, pos_dev, M_dev, M, d, emb_scale, E, pe, g, b,
                                                            x, y);
  }
  // M is the row count, or its upper bound when M_dev supplies it on device
  void embed_ln(const int* ids, const int* pos, int pos_const, int M, const float* g, const float* b, float* x, T* y,
                const int* pos_dev = nullptr, const int* M_dev = nullptr) {
    if (M <= 0) return;
    Scope sc(this, K_OTHER, (double)M * d * (4 + 4 + 2 * sizeof(T)), 8.0 * M * d);
    const int npl = cdiv(d, 32);
#define HRT_EMB(N) emb_launch<N>(ids, pos, pos_const, pos_dev, M_dev, M, g, b, x, y)
    if (npl <= 1) HRT_EMB(1);
    else if (npl <= 2) HRT_EMB(2);
    else if (npl <= 4) HRT_EMB(4);
    else if (npl <= 8) HRT_EMB(8);
    else if (npl <= 16) HRT_EMB(16);
    else HRT_EMB(32);
#undef HRT_EMB
    check_launch();
  }

  // ragged whole-sequence attention (see attn_prefill_kernel)
  template <int DH>
  void prefill_launch(dim3 grid, const int2* items, const T* q, int qs, const T* k, const T* v, int kvs, T* out,
                      int os, const int* q_off, const int* q_slot, const int* q_len, const int* kv_map,
                      const int* kv_off, const int* kv_len, const unsigned char* key_ok, int causal) {
    launch(attn_prefill_kernel<T, DH>, grid, AP_WARPS * 32, 0, items, q, qs, k, v, kvs, out, os, q_off, q_slot,
                                                                   q_len, kv_map, kv_off, kv_len, key_ok, causal,
                                                                   att_scale);
  }
  // work items (sequence, 32-query block) for every sequence with slot rows
  static std::vector<int> prefill_items(const std::vector<int>& slot) {
    std::vector<int> it;
    for (size_t s = 0; s < slot.size(); ++s)
      for (int b = 0; b * 32 < slot[s]; ++b) {
        it.push_back((int)s);
        it.push_back(b);
      }
    return it;
  }
  void attn_prefill(const int* items, int n_items, const T* q, int qs, const T* k, const T* v, int kvs, T* out,
                    int os, const int* q_off, const int* q_slot, const int* q_len, const int* kv_map,
                    const int* kv_off, const int* kv_len, const unsigned char* key_ok, int causal, double flops) {
    if (n_items <= 0) return;
    Scope sc(this, K_ATTN, 0.0, flops);
    dim3 grid(n_items, H);
    const int2* it2 = reinterpret_cast<const int2*>(items);
#define HRT_PF(DHV) prefill_launch<DHV>(grid, it2, q, qs, k, v, kvs, out, os, q_off, q_slot, q_len, kv_map, kv_off, kv_len, key_ok, causal)
    if constexpr (BF16) {
      // all heads per CTA (K/V rows fetched once); with few work items per-head CTAs spread wider
      if (dh == 64 && (H == 1 || H == 2 || H == 4 || H == 8) &&
          (attn_heads_mode == 2 || (attn_heads_mode == 1 && n_items >= num_sms))) {
        // heads per CTA: all (K / V rows fetched once), or H / attn_head_groups (smaller CTAs,
        // more of them resident per SM)
        const int ht = std::max(1, H / std::max(1, attn_head_groups));
        const size_t smem = attn_heads_smem(ht * dh);
        auto go = [&](auto kern) {
          smem_optin(kern, smem);
          launch(kern, dim3(n_items, H / ht), 2 * ht * 32, smem, it2, q, qs, k, v, kvs, out, os, q_off, q_slot, q_len,
                 kv_map, kv_off, kv_len, key_ok, causal, att_scale, H);
        };
        if (ht == 8)
          go(attn_prefill_heads_kernel<8>);
        else if (ht == 4)
          go(attn_prefill_heads_kernel<4>);
        else if (ht == 2)
          go(attn_prefill_heads_kernel<2>);
        else
          go(attn_prefill_heads_kernel<1>);
        check_launch();
        return;
      }
      if (dh == 64) {
        launch(attn_prefill_mma_kernel, grid, AM_WARPS * 32, 0, it2, q, qs, k, v, kvs, out, os, q_off, q_slot,
                                                                   q_len, kv_map, kv_off, kv_len, key_ok, causal,
                                                                   att_scale);
        check_launch();
        return;
      }
    }
    switch (dh) {
      case 8: HRT_PF(8); break;
      case 16: HRT_PF(16); break;
      case 32: HRT_PF(32); break;
      case 64: HRT_PF(64); break;
      default: throw HrtError(HRT_ERR_INVALID, "d_head must be 8, 16, 32 or 64");
    }
#undef HRT_PF
    check_launch();
  }

  template <int DH, bool SELF>
  void decode_launch(int blocks, size_t smem, const T* q, int qs, const T* kn, const T* vn, int ns, T* kc, T* vc,
                     const int* hist, const int* hist2, int cap, int t, const int* t_dev, const int* row_seq,
                     const int* kv_off, const int* kv_len, const int* R_dev, int R, int lk_max, T* out) {
    launch(attn_decode_kernel<T, DH, SELF>, blocks, 128, smem, q, qs, kn, vn, ns, kc, vc, d, hist, hist2, cap, t, t_dev,
                                                                  row_seq, kv_off, kv_len, R_dev, R, H, lk_max,
                                                                  att_scale, out, d, cross_prefetch ? 1 : 0);
  }
  template <bool SELF>
  void attn_decode(const T* q, int qs, const T* kn, const T* vn, int ns, T* kc, T* vc, const int* hist, int cap, int t,
                   const int* row_seq, const int* kv_off, const int* kv_len, int R, int lk_max, T* out,
                   double bytes, const int* t_dev = nullptr, const int* R_dev = nullptr, const int* hist2 = nullptr) {
    if (R <= 0) return;
    Scope sc(this, K_ATTN, bytes, 0.0);
    // debug option "attn_pdl" = 0: decode attention launched without the programmatic edge
    struct PdlScope {
      bool& f;
      bool old;
      PdlScope(bool& flag, bool v) : f(flag), old(flag) { f = v; }
      ~PdlScope() { f = old; }
    } pdl_scope(pdl, pdl && attn_pdl);
    if constexpr (BF16) {
      // large row counts only (few rows: the warp-per-(row, head) kernel spreads wider); the
      // choice follows the graph's row bucket so graph and eager runs match bit for bit
      const int Rp = path_rows > 0 ? path_rows : R;
      if (dh == 64 && (H == 1 || H == 2 || H == 4 || H == 8 || H == 16) &&
          (attn_rows_mode == 2 || (attn_rows_mode == 1 && Rp >= 256))) {
        // one CTA per row, all heads: coalesced whole-row K/V staging
        const size_t smem = attn_rows_smem(d);
        const int threads = std::max(64, H * 32);
        auto go = [&](auto kern) {
          smem_optin(kern, smem);
          launch(kern, R, threads, smem, q, qs, kn, vn, ns, kc, vc, d, greedy_hist_identity ? nullptr : hist,
                 greedy_hist_identity ? nullptr : hist2, cap, t, t_dev, row_seq, kv_off, kv_len, R_dev, R, H, att_scale,
                 out, d, cross_prefetch ? 1 : 0);
        };
        if (H == 8)
          go(attn_decode_rows_kernel<SELF, 8>);
        else if (H == 16)
          go(attn_decode_rows_kernel<SELF, 16>);
        else if (H == 4)
          go(attn_decode_rows_kernel<SELF, 4>);
        else if (H == 2)
          go(attn_decode_rows_kernel<SELF, 2>);
        else
          go(attn_decode_rows_kernel<SELF, 1>);
        check_launch();
        return;
      }
    }
    if (greedy_hist_identity) {  // greedy: slot j of row r is row r (no history lookups)
      hist = nullptr;
      hist2 = nullptr;
    }
    const int nwarp = 4;
    lk_max = std::max(lk_max, 1);
    const size_t smem = (size_t)nwarp * lk_max * sizeof(float);
    const int blocks = cdiv(R * H, nwarp);
#define HRT_DC(DHV) decode_launch<DHV, SELF>(blocks, smem, q, qs, kn, vn, ns, kc, vc, hist, hist2, cap, t, t_dev, row_seq, kv_off, kv_len, R_dev, R, lk_max, out)
    switch (dh) {
      case 8: HRT_DC(8); break;
      case 16: HRT_DC(16); break;
      case 32: HRT_DC(32); break;
      case 64: HRT_DC(64); break;
      default: throw HrtError(HRT_ERR_INVALID, "d_head must be 8, 16, 32 or 64");
    }
#undef HRT_DC
    check_launch();
  }

  // vocab projection of R rows of y (K-major d) into tile partials.
  // ln_g != nullptr: the rows are LN(s1.x) with the final decoder LayerNorm
  // (dec_lng / dec_lnb), computed in the GEMV prologue
  void vocab_parts(const T* y, int y_cap, int R, VocabParts& parts, int kt, int norm_allowed, float* logits_buf,
                   const int* M_dev = nullptr, const float* ln_g = nullptr) {
    if (R <= 0) return;
    if constexpr (BF16) {
      if ((kt == 1 || (kt <= 5 && !ln_g)) && gemv_vocab_ok(R)) {
        parts.ntiles = cdiv(V, GV_VTILE);
        Scope sc(this, K_VOCAB | K_GEMM, 2.0 * ((double)V * d + (double)R * d), 2.0 * R * (double)V * d);
        const bf16* yb = reinterpret_cast<const bf16*>(y);
        const bf16* Eb = reinterpret_cast<const bf16*>(frag_of(E));
        const GvLN ln{ln_g ? s1.x : nullptr, dec_lng, dec_lnb};
        const int grid = cdiv(V, GV_VTILE);
#define HRT_GVV(NT)                                                                                          \
  do {                                                                                                       \
    if (kt > 1)                                                                                              \
      launch(gemv_vocab_kernel<NT, false, 5>, grid, GV_VWARPS * 32, 0, yb, d, Eb, V, d, R, M_dev, parts, norm_allowed, ln); \
    else if (ln_g)                                                                                           \
      launch(gemv_vocab_kernel<NT, true>, grid, GV_VWARPS * 32, 0, yb, d, Eb, V, d, R, M_dev, parts, norm_allowed, ln); \
    else                                                                                                     \
      launch(gemv_vocab_kernel<NT, false>, grid, GV_VWARPS * 32, 0, yb, d, Eb, V, d, R, M_dev, parts, norm_allowed, ln); \
  } while (0)
        if (R <= 8)
          HRT_GVV(1);
        else if (R <= 16)
          HRT_GVV(2);
        else
          HRT_GVV(4);
#undef HRT_GVV
        check_launch();
        return;
      }
      if (ln_g) {  // tcgen05 path: unfused final LN
        layernorm(s1.x, R, dec_lng, dec_lnb, const_cast<T*>(y), nullptr, nullptr, M_dev);
      }
      const int bn = vocab_bn(R);
      parts.ntiles = cdiv(V, bn / 2);  // one partial per epilogue column half
      Scope sc(this, K_VOCAB | K_GEMM, 2.0 * ((double)V * d + (double)R * d), 2.0 * R * (double)V * d);
      if (kt == 1) {
        VocabEpi<1> epi{parts, norm_allowed, bn / 2};
        launch_vocab(y, y_cap, R, epi, bn, M_dev);
      } else if (kt <= 5) {
        VocabEpi<5> epi{parts, norm_allowed, bn / 2};
        launch_vocab(y, y_cap, R, epi, bn, M_dev);
      } else {
        VocabEpi<KTOP_MAX> epi{parts, norm_allowed, bn / 2};
        launch_vocab(y, y_cap, R, epi, bn, M_dev);
      }
      check_launch();
    } else {
      if (M_dev) throw HrtError(HRT_ERR_INVALID, "device row count unsupported on the fp32 vocab path");
      // fp32: materialise logits in row blocks, then reduce per 256-col tile
      parts.ntiles = cdiv(V, 256);
      for (int r0 = 0; r0 < R; r0 += logit_rows) {
        const int rn = std::min(logit_rows, R - r0);
        {
          Scope sc(this, K_VOCAB | K_GEMM, 4.0 * ((double)V * d + (double)rn * d + (double)rn * V),
                   2.0 * rn * (double)V * d);
          EpiStoreF32 epi{logits_buf, V};
          if (!gemv_f32(y + (size_t)r0 * d, d, E, V, d, rn, rn, nullptr, epi)) {
            dim3 grid(cdiv(V, SG_BN), cdiv(rn, SG_BM));
            launch(simt_gemm_kernel<T, EpiStoreF32>, grid, SG_THREADS, 0, y + (size_t)r0 * d, d, E, d, rn, V, d,
                                                                              nullptr, epi, V % 4 == 0);
          }
          check_launch();
        }
        VocabParts sub = parts;
        sub.mx += (size_t)r0 * parts.ntiles;
        sub.sum += (size_t)r0 * parts.ntiles;
        sub.val += (size_t)r0 * parts.ntiles * kt;
        sub.id += (size_t)r0 * parts.ntiles * kt;
        sub.eos += r0;
        Scope sc(this, K_OTHER, 4.0 * rn * V, 0);
        dim3 grid(rn, parts.ntiles);
        if (kt == 1)
          launch(rowstats_from_logits_kernel<1>, grid, 32, 0, logits_buf, V, V, nullptr, sub, 256, norm_allowed);
        else if (kt <= 5)
          launch(rowstats_from_logits_kernel<5>, grid, 32, 0, logits_buf, V, V, nullptr, sub, 256, norm_allowed);
        else
          launch(rowstats_from_logits_kernel<KTOP_MAX>, grid, 32, 0, logits_buf, V, V, nullptr, sub, 256,
                 norm_allowed);
        check_launch();
      }
    }
  }
  template <class Epi>
  void launch_vocab(const T* y, int y_cap, int R, const Epi& epi, int bn, const int* M_dev = nullptr) {
    if (bn == 64)
      tc_launch<64, 8>(y, y_cap, d, R, E, V, d, epi, M_dev);
    else if (bn == 128)
      tc_launch<128, 6>(y, y_cap, d, R, E, V, d, epi, M_dev);
    else
      tc_launch<256, 4>(y, y_cap, d, R, E, V, d, epi, M_dev);
  }

  // full fp32 logits of R rows (protocol face / parity), chunked
  void full_logits(const T* y, int y_cap, int R, float* dst) {
    Scope sc(this, K_VOCAB | K_GEMM, sizeof(T) * ((double)V * d + (double)R * d), 2.0 * R * (double)V * d);
    EpiStoreF32 epi{dst, V};
    if constexpr (BF16) {
      launch_vocab(y, y_cap, R, epi, choose_bn(R, V));
    } else {
      dim3 grid(cdiv(V, SG_BN), cdiv(R, SG_BM));
      launch(simt_gemm_kernel<T, EpiStoreF32>, grid, SG_THREADS, 0, y, d, E, d, R, V, d, nullptr, epi, V % 4 == 0);
    }
    check_launch();
  }

  // -------------------------------------------------------------------------
  // phase 1: encoder over packed sources (infer.py:176-221), then the fused
  // cross-K/V projection of every decoder layer (infer.py:216-220).
  // d_ids / d_pos hold the packed tokens; seq metadata in device arrays.
  // -------------------------------------------------------------------------
  void run_encoder(int M, int nseq, int max_len_seq, const int* off, const int* len, const int* items, int n_items) {
    Tag _tg(this, "encoder");
    if (M > Me_max) throw HrtError(HRT_ERR_MEMORY, "encoder tokens exceed max_src_tokens");
    if (Le > 0)
      embed_ln(d_ids, d_pos, 0, M, enc[0].ln1g, enc[0].ln1b, eb.x, eb.y);
    else
      embed_ln(d_ids, d_pos, 0, M, enc_lng, enc_lnb, eb.x, eb.y);
    const int sk = enc_skip;  // debug attribution: 1 LN, 2 attention, 4 projections (wrong results)
    for (int i = 0; i < Le; ++i) {
      const EncW& w = enc[i];
      if (!(sk & 4)) {
        Tag _t(this, "encoder.qkv");
        gemm(K_GEMM, eb.y, Me_max, d, M, w.wqkv, 3 * d, d, EpiBiasT<T, false>{eb.qkv, 3 * d, w.bqkv});
      }
      Tag _ta(this, "encoder.attn");
      if (!(sk & 2))
        attn_prefill(items, n_items, eb.qkv, 3 * d, eb.qkv + d, eb.qkv + 2 * d, 3 * d, eb.ctx, d, off, len, len,
                     nullptr, off, len, nullptr, 0, 4.0 * d * (double)max_len_seq * M);
      // residual projections carry the next LayerNorm (fused epilogue on the tcgen05 path)
      const float* ng = i + 1 < Le ? enc[i + 1].ln1g : enc_lng;
      const float* nb = i + 1 < Le ? enc[i + 1].ln1b : enc_lnb;
      if (sk == 0) {
        {
          Tag _t(this, "encoder.wo+ln");
          gemm_res_ln(eb.ctx, Me_max, d, M, w.wo, d, eb.x, w.bo, w.ln2g, w.ln2b, eb.y, nullptr);
        }
        {
          Tag _t(this, "encoder.w1");
          gemm(K_GEMM, eb.y, Me_max, d, M, w.w1, ff, d, EpiBiasT<T, true>{eb.hid, ff, w.b1});
        }
        if (i + 1 < Le || !p_mem_target) {
          Tag _t(this, "encoder.w2+ln");
          gemm_res_ln(eb.hid, Me_max, ff, M, w.w2, ff, eb.x, w.b2, ng, nb, eb.y, nullptr);
        } else {  // protocol encode: the final LN also writes the fp32 memory
          gemm(K_GEMM, eb.hid, Me_max, ff, M, w.w2, d, ff, EpiResidual{eb.x, d, w.b2});
          layernorm(eb.x, M, enc_lng, enc_lnb, eb.y, nullptr, p_mem_target);
        }
        continue;
      }
      if (!(sk & 4)) gemm(K_GEMM, eb.ctx, Me_max, d, M, w.wo, d, d, EpiResidual{eb.x, d, w.bo});
      if (!(sk & 1)) layernorm(eb.x, M, w.ln2g, w.ln2b, eb.y);
      if (!(sk & 4)) gemm(K_GEMM, eb.y, Me_max, d, M, w.w1, ff, d, EpiBiasT<T, true>{eb.hid, ff, w.b1});
      if (!(sk & 4)) gemm(K_GEMM, eb.hid, Me_max, ff, M, w.w2, d, ff, EpiResidual{eb.x, d, w.b2});
      if (!(sk & 1) || i + 1 == Le) layernorm(eb.x, M, ng, nb, eb.y, nullptr, i + 1 < Le ? nullptr : p_mem_target);
    }
    gemm(K_GEMM, eb.y, Me_max, d, M, wxkv, Ld * 2 * d, d, EpiBiasT<T, false>{xkv, Ld * 2 * d, bxkv});
  }
  float* p_mem_target = nullptr;

  // -------------------------------------------------------------------------
  // one Stage-I decoder call for rows 0..R-1 at position `pos`, cache slot t
  // (infer.py:234-301 up to the final LN; vocab handled by the caller)
  // -------------------------------------------------------------------------
  // ctl != nullptr: graph mode -- R is the upper bound (grid sizing) and the
  // live row count, step and position are read from the device control block.
  void decoder_step(int R, int t, int pos, int cap, const int* feed, const int* hist, const int* row_seq,
                    const int* kv_off, const int* kv_len, int max_src, StepCtl* ctl = nullptr,
                    bool do_embed = true, const int* hist2 = nullptr, bool final_ln_fused = false) {
    const int* Rd = ctl ? &ctl->R : nullptr;
    const int* td = ctl ? &ctl->t : nullptr;
    Tag _tg4(this, "s1.embed_ln");
    if (do_embed && !(s1_skip & 32)) embed_ln(feed, nullptr, pos, R, dec[0].ln1g, dec[0].ln1b, s1.x, s1.y, ctl ? &ctl->pos : nullptr, Rd);
    for (int i = 0; i < Ld; ++i) {
      const DecW& w = dec[i];
      T* kc = s1.kc + (size_t)i * R_max * cap_max * d;
      T* vc = s1.vc + (size_t)i * R_max * cap_max * d;
      Tag _tg10(this, "s1.qkv");
      if (!(s1_skip & 4)) gemm(K_GEMM, s1.y, R_max, d, R, w.wqkv, 3 * d, d, EpiBiasT<T, false>{s1.qkv, 3 * d, w.bqkv}, Rd);
      Tag _tg12(this, "s1.attn_self");
      if (!(s1_skip & 66)) attn_decode<true>(s1.qkv, 3 * d, s1.qkv + d, s1.qkv + 2 * d, 3 * d, kc, vc, hist, cap, t, nullptr, nullptr,
                        nullptr, R, cap, s1.ctx, 2.0 * sizeof(T) * (double)R * (t + 1) * d, td, Rd, hist2);
      // Wo + residual (+ LN2 in the GEMV tail on the small-row path)
      // the LayerNorm after each residual projection rides in its epilogue: GEMV tail
      // (option tail_ln) or the tcgen05 cluster epilogue (option ln_epi, rows above the GEMV regime)
      const bool tail = (tail_ln_ok(R, d) || ln_epi_ok(R, d)) && !(s1_skip & 5);
      Tag _tg15(this, "s1.wo");
      if (tail)
        gemm_res_ln(s1.ctx, R_max, d, R, w.wo, d, s1.x, w.bo, w.ln2g, w.ln2b, s1.y, Rd);
      else if (!(s1_skip & 4))
        gemm(K_GEMM, s1.ctx, R_max, d, R, w.wo, d, d, EpiResidual{s1.x, d, w.bo}, Rd);
      Tag _tg19(this, "s1.qc");
      if (tail)
        gemm(K_GEMM, s1.y, R_max, d, R, w.wqc, d, d, EpiBiasT<T, false>{s1.qc, d, w.bqc}, Rd);
      else if (!(s1_skip & 4))
        gemm_ln(K_GEMM, s1.x, w.ln2g, w.ln2b, s1.y, R_max, R, w.wqc, d, EpiBiasT<T, false>{s1.qc, d, w.bqc}, Rd);
      Tag _tg21(this, "s1.attn_cross");
      if (!(s1_skip & 130)) attn_decode<false>(s1.qc, d, xkv + (size_t)2 * i * d, xkv + (size_t)(2 * i + 1) * d, Ld * 2 * d, nullptr,
                         nullptr, nullptr, 0, 0, row_seq, kv_off, kv_len, R, max_src, s1.ctx,
                         2.0 * sizeof(T) * (double)R * max_src * d, nullptr, Rd);
      Tag _tg25(this, "s1.woc");
      if (tail)
        gemm_res_ln(s1.ctx, R_max, d, R, w.woc, d, s1.x, w.boc, w.ln3g, w.ln3b, s1.y, Rd);
      else if (!(s1_skip & 4))
        gemm(K_GEMM, s1.ctx, R_max, d, R, w.woc, d, d, EpiResidual{s1.x, d, w.boc}, Rd);
      Tag _tg29(this, "s1.w1");
      if (tail)
        gemm(K_GEMM, s1.y, R_max, d, R, w.w1, ff, d, EpiBiasT<T, true>{s1.hid, ff, w.b1}, Rd);
      else if (!(s1_skip & 4))
        gemm_ln(K_GEMM, s1.x, w.ln3g, w.ln3b, s1.y, R_max, R, w.w1, ff, EpiBiasT<T, true>{s1.hid, ff, w.b1}, Rd);
      // W2 + residual (+ the next LayerNorm: next layer's LN1 or the final LN)
      const float* ng = i + 1 < Ld ? dec[i + 1].ln1g : dec_lng;
      const float* nb = i + 1 < Ld ? dec[i + 1].ln1b : dec_lnb;
      const bool tail2 = tail && (tail_ln_ok(R, ff) || ln_epi_ok(R, ff)) && !(i + 1 == Ld && final_ln_fused);
      Tag _tg31(this, "s1.w2");
      if (tail2)
        gemm_res_ln(s1.hid, R_max, ff, R, w.w2, ff, s1.x, w.b2, ng, nb, s1.y, Rd);
      else if (!(s1_skip & 4))
        gemm(K_GEMM, s1.hid, R_max, ff, R, w.w2, d, ff, EpiResidual{s1.x, d, w.b2}, Rd);
      Tag _tg34(this, "s1.ln_out");
      if (s1_skip & 1 || tail2) {
      } else if (i + 1 < Ld)
        layernorm(s1.x, R, dec[i + 1].ln1g, dec[i + 1].ln1b, s1.y, nullptr, nullptr, Rd);
      else if (!final_ln_fused)
        layernorm(s1.x, R, dec_lng, dec_lnb, s1.y, nullptr, nullptr, Rd);
    }
  }

  // -------------------------------------------------------------------------
  // one parallel (Stage-II) decoder pass over packed candidate slots
  // (infer.py:322-396). Leaves the final-LN'd rows in s2.y (or, with
  // out_row, gathered into s2.ymask).
  // -------------------------------------------------------------------------
  void decoder_parallel(int M2, int nc, int max_slot, int max_src, const int* off, const int* slot,
                        const int* qlen, const int* kv_map, const int* src_off, const int* src_len,
                        const unsigned char* key_ok, int causal, const int* out_row, const int* items, int n_items) {
    Tag _tg(this, "stage2.decoder");
    embed_ln(s2.ids, s2.pos, 0, M2, dec[0].ln1g, dec[0].ln1b, s2.x, s2.y);
    for (int i = 0; i < Ld; ++i) {
      const DecW& w = dec[i];
      gemm(K_GEMM, s2.y, M2_max, d, M2, w.wqkv, 3 * d, d, EpiBiasT<T, false>{s2.qkv, 3 * d, w.bqkv});
      attn_prefill(items, n_items, s2.qkv, 3 * d, s2.qkv + d, s2.qkv + 2 * d, 3 * d, s2.ctx, d, off, slot, qlen,
                   nullptr, off, qlen, key_ok, causal, 4.0 * d * (double)max_slot * M2);
      gemm_res_ln(s2.ctx, M2_max, d, M2, w.wo, d, s2.x, w.bo, w.ln2g, w.ln2b, s2.y, nullptr);
      gemm(K_GEMM, s2.y, M2_max, d, M2, w.wqc, d, d, EpiBiasT<T, false>{s2.qc, d, w.bqc});
      attn_prefill(items, n_items, s2.qc, d, xkv + (size_t)2 * i * d, xkv + (size_t)(2 * i + 1) * d, Ld * 2 * d,
                   s2.ctx, d, off, slot, qlen, kv_map, src_off, src_len, nullptr, 0, 4.0 * d * (double)max_src * M2);
      gemm_res_ln(s2.ctx, M2_max, d, M2, w.woc, d, s2.x, w.boc, w.ln3g, w.ln3b, s2.y, nullptr);
      gemm(K_GEMM, s2.y, M2_max, d, M2, w.w1, ff, d, EpiBiasT<T, true>{s2.hid, ff, w.b1});
      if (i + 1 < Ld)
        gemm_res_ln(s2.hid, M2_max, ff, M2, w.w2, ff, s2.x, w.b2, dec[i + 1].ln1g, dec[i + 1].ln1b, s2.y, nullptr);
      else if (out_row)  // only the [MASK] rows are normalised, gathered into the vocab operand
        gemm_res_ln(s2.hid, M2_max, ff, M2, w.w2, ff, s2.x, w.b2, dec_lng, dec_lnb, s2.ymask, nullptr, out_row);
      else
        gemm_res_ln(s2.hid, M2_max, ff, M2, w.w2, ff, s2.x, w.b2, dec_lng, dec_lnb, s2.y, nullptr);
    }
  }

  // metadata upload: host vector -> d_meta (one H2D copy), returns device ptrs
  int* meta_put(size_t& cursor, const std::vector<int>& v) {
    const size_t o = cursor;
    if (o + v.size() > (size_t)meta_cap) throw HrtError(HRT_ERR_MEMORY, "metadata buffer overflow");
    std::copy(v.begin(), v.end(), h_meta + o);
    cursor += v.size();
    cursor = (cursor + 7) & ~size_t(7);
    return d_meta + o;
  }
  void meta_flush(size_t cursor) {
    // the fixed header (Stage-I control) is copied with the call's metadata
    CUDA_OK(cudaMemcpyAsync(d_meta, h_meta, cursor * sizeof(int), cudaMemcpyHostToDevice, stream));
    CUDA_OK(cudaEventRecord(meta_ev, stream));
  }
  // the previous call's metadata copy must have left the pinned buffer
  void meta_reset() { CUDA_OK(cudaEventSynchronize(meta_ev)); }

  // -------------------------------------------------------------------------
  // session protocol
  // -------------------------------------------------------------------------
  void encode(const int32_t* ids, const int32_t* lens, int n, float* mem_out) override {
    if (n < 1) throw HrtError(HRT_ERR_INVALID, "n_seq out of range");
    if (n > Bmax) throw HrtError(HRT_ERR_MEMORY, "n_seq exceeds the arena's max_sentences");
    std::vector<int> off(n + 1, 0), len(n);
    int maxl = 0;
    for (int i = 0; i < n; ++i) {
      if (lens[i] < 1) throw HrtError(HRT_ERR_INFERENCE, "empty source");
      if (lens[i] > Lmax)
        throw HrtError(HRT_ERR_INFERENCE, "source length " + std::to_string(lens[i]) + " exceeds max_len " +
                                              std::to_string(Lmax));
      len[i] = lens[i];
      off[i + 1] = off[i] + lens[i];
      maxl = std::max(maxl, lens[i]);
    }
    const int M = off[n];
    if (M > Me_max) throw HrtError(HRT_ERR_MEMORY, "encoder tokens exceed capacity");
    for (int i = 0; i < M; ++i)
      if (ids[i] < 0 || ids[i] >= V) throw HrtError(HRT_ERR_INVALID, "source token id out of range");
    std::vector<int> pos(M);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < len[i]; ++j) pos[off[i] + j] = j;
    meta_reset();
    size_t cur = meta_hdr;
    int* d_off = meta_put(cur, off);
    int* d_len = meta_put(cur, len);
    const std::vector<int> items = prefill_items(len);
    int* d_items = meta_put(cur, items);
    meta_flush(cur);
    CUDA_OK(cudaMemcpyAsync(d_ids, ids, M * sizeof(int), cudaMemcpyHostToDevice, stream));
    CUDA_OK(cudaMemcpyAsync(d_pos, pos.data(), M * sizeof(int), cudaMemcpyHostToDevice, stream));
    // keep encoded-sequence metadata on device for later protocol calls
    p_seq_off = off;
    p_seq_len = len;
    p_nseq = n;
    if (mem_out) {
      if (p_mem_cap < (size_t)M * d) {
        cudaFree(p_mem);
        CUDA_OK(cudaMalloc(&p_mem, (size_t)M * d * sizeof(float)));
        p_mem_cap = (size_t)M * d;
      }
      p_mem_target = p_mem;
    }
    run_encoder(M, n, maxl, d_off, d_len, d_items, (int)items.size() / 2);
    note_high_water(0, ArenaDims{M, 0, 0, 0});
    p_mem_target = nullptr;
    if (Le == 0 && mem_out) throw HrtError(HRT_ERR_INVALID, "memory output needs enc_layers >= 1");
    if (mem_out) {
      CUDA_OK(cudaMemcpyAsync(mem_out, p_mem, (size_t)M * d * sizeof(float), cudaMemcpyDeviceToHost, stream));
    }
    CUDA_OK(cudaStreamSynchronize(stream));
    p_has_cache = false;
  }

  // device copies of encoded-sequence metadata for protocol calls
  int *p_doff = nullptr, *p_dlen = nullptr;
  void upload_seq_meta(size_t& cur, std::vector<int>& extra_unused) {
    (void)extra_unused;
    p_doff = meta_put(cur, p_seq_off);
    p_dlen = meta_put(cur, p_seq_len);
  }

  std::vector<int> p_rowseq_h;
  void start_cache(int rows, int cap, const int32_t* row_seq) override {
    if (p_nseq == 0) throw HrtError(HRT_ERR_INFERENCE, "encode() must precede start_cache()");
    if (rows < 1) throw HrtError(HRT_ERR_INVALID, "rows out of range");
    if (rows > R_max) throw HrtError(HRT_ERR_MEMORY, "rows exceed the arena's max_sentences * max_beam");
    if (cap < 1 || cap > cap_max) throw HrtError(HRT_ERR_INVALID, "cache capacity out of range");
    p_rows = rows;
    p_cap = cap;
    note_high_water(1, ArenaDims{0, rows, 0, 0});
    p_len = 0;
    p_last_pos = -1;
    p_has_cache = true;
    p_rowseq_h.assign(rows, 0);
    if (row_seq)
      for (int r = 0; r < rows; ++r) {
        if (row_seq[r] < 0 || row_seq[r] >= p_nseq) throw HrtError(HRT_ERR_INVALID, "row_seq out of range");
        p_rowseq_h[r] = row_seq[r];
      }
    CUDA_OK(cudaMemcpyAsync(s_rowseq, p_rowseq_h.data(), rows * sizeof(int), cudaMemcpyHostToDevice, stream));
    launch(stage1_init_kernel, cdiv(rows, 128), 128, 0, rows, cap, BOS_ID, s_feed, s_done, s_nsteps, s_forced,
                                                           s_score, s_hist);
    check_launch();
    stats.kernel_launches++;
  }

  void step(const int32_t* tokens, int position, float* logp_out) override {
    if (!p_has_cache) throw HrtError(HRT_ERR_INFERENCE, "start_cache() must precede step()");
    if (p_last_pos >= 0 && position <= p_last_pos)
      throw HrtError(HRT_ERR_INFERENCE, "new position must exceed all cached positions");
    if (p_len >= p_cap) throw HrtError(HRT_ERR_INFERENCE, "decoder cache capacity exceeded");
    if (position < 0 || position >= P) throw HrtError(HRT_ERR_INFERENCE, "position exceeds the positional table");
    for (int r = 0; r < p_rows; ++r)
      if (tokens[r] < 0 || tokens[r] >= V) throw HrtError(HRT_ERR_INVALID, "token id out of range");
    meta_reset();
    size_t cur = meta_hdr;
    std::vector<int> dummy;
    upload_seq_meta(cur, dummy);
    meta_flush(cur);
    CUDA_OK(cudaMemcpyAsync(s_feed, tokens, p_rows * sizeof(int), cudaMemcpyHostToDevice, stream));
    int max_src = *std::max_element(p_seq_len.begin(), p_seq_len.end());
    decoder_step(p_rows, p_len, position, p_cap, s_feed, s_hist, s_rowseq, p_doff, p_dlen, max_src);
    if (logp_out) {
      for (int r0 = 0; r0 < p_rows; r0 += logit_rows) {
        const int rn = std::min(logit_rows, p_rows - r0);
        full_logits(s1.y + (size_t)r0 * d, R_max - r0, rn, s1.logits);
        launch(logsoftmax_rows_kernel, rn, 256, 0, s1.logits, V, V);
        check_launch();
        stats.kernel_launches++;
        CUDA_OK(cudaMemcpyAsync(logp_out + (size_t)r0 * V, s1.logits, (size_t)rn * V * sizeof(float),
                                cudaMemcpyDeviceToHost, stream));
      }
    }
    CUDA_OK(cudaStreamSynchronize(stream));
    p_len += 1;
    p_last_pos = position;
    stats.decoder_calls += 1;
  }

  void reorder(const int32_t* parents) override {
    if (!p_has_cache) throw HrtError(HRT_ERR_INFERENCE, "start_cache() must precede reorder()");
    bool ident = true;
    for (int r = 0; r < p_rows; ++r) {
      if (parents[r] < 0 || parents[r] >= p_rows) throw HrtError(HRT_ERR_INVALID, "parent row out of range");
      ident &= parents[r] == r;
    }
    if (ident) return;
    CUDA_OK(cudaMemcpyAsync(s_parents, parents, p_rows * sizeof(int), cudaMemcpyHostToDevice, stream));
    launch(reorder_hist_kernel, p_rows, 128, 0, s_parents, s_hist, s_hist2, p_rows, p_cap, p_len);
    check_launch();
    stats.kernel_launches++;
    std::swap(s_hist, s_hist2);
    CUDA_OK(cudaStreamSynchronize(stream));
  }

  void parallel_logits(const int32_t* ids, const int32_t* pos, const uint8_t* pad, int B, int Tn, int mode,
                       const int32_t* seq, float* logits_out) override {
    if (p_nseq == 0) throw HrtError(HRT_ERR_INFERENCE, "encode() must precede parallel_logits()");
    if (B < 1 || Tn < 1) throw HrtError(HRT_ERR_INVALID, "empty parallel batch");
    if (mode != 0 && mode != 1) throw HrtError(HRT_ERR_INFERENCE, "unknown mode");
    const int M2 = B * Tn;
    if (M2 > M2_max) throw HrtError(HRT_ERR_MEMORY, "parallel batch exceeds capacity");
    for (int i = 0; i < M2; ++i) {
      if (pos[i] < 0 || pos[i] >= P) throw HrtError(HRT_ERR_INVALID, "position exceeds the positional table");
      if (ids[i] < 0 || ids[i] >= V) throw HrtError(HRT_ERR_INVALID, "token id out of range");
    }
    std::vector<int> off(B + 1), slot(B, Tn), qlen(B, Tn), kvmap(B, 0);
    for (int b = 0; b <= B; ++b) off[b] = b * Tn;
    if (seq)
      for (int b = 0; b < B; ++b) {
        if (seq[b] < 0 || seq[b] >= p_nseq) throw HrtError(HRT_ERR_INVALID, "seq out of range");
        kvmap[b] = seq[b];
      }
    meta_reset();
    size_t cur = meta_hdr;
    int* d_off = meta_put(cur, off);
    int* d_slot = meta_put(cur, slot);
    int* d_qlen = meta_put(cur, qlen);
    int* d_map = meta_put(cur, kvmap);
    const std::vector<int> items = prefill_items(slot);
    int* d_items = meta_put(cur, items);
    std::vector<int> dummy;
    upload_seq_meta(cur, dummy);
    // key mask bytes packed into ints region
    unsigned char* d_keyok = nullptr;
    if (pad) {
      std::vector<int> packed((M2 + 3) / 4, 0);
      std::memcpy(packed.data(), pad, M2);
      d_keyok = reinterpret_cast<unsigned char*>(meta_put(cur, packed));
    }
    meta_flush(cur);
    CUDA_OK(cudaMemcpyAsync(s2.ids, ids, M2 * sizeof(int), cudaMemcpyHostToDevice, stream));
    CUDA_OK(cudaMemcpyAsync(s2.pos, pos, M2 * sizeof(int), cudaMemcpyHostToDevice, stream));
    int max_src = *std::max_element(p_seq_len.begin(), p_seq_len.end());
    decoder_parallel(M2, B, Tn, max_src, d_off, d_slot, d_qlen, d_map, p_doff, p_dlen, d_keyok, mode, nullptr, d_items,
                     (int)items.size() / 2);
    note_high_water(2, ArenaDims{0, 0, M2, 0});
    if (p_logits_cap < (size_t)M2 * V) {
      cudaFree(p_logits);
      CUDA_OK(cudaMalloc(&p_logits, (size_t)M2 * V * sizeof(float)));
      p_logits_cap = (size_t)M2 * V;
    }
    full_logits(s2.y, M2_max, M2, p_logits);
    if (logits_out)
      CUDA_OK(cudaMemcpyAsync(logits_out, p_logits, (size_t)M2 * V * sizeof(float), cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaStreamSynchronize(stream));
    p_B = B;
    p_T = Tn;
    stats.decoder_calls += 1;
  }

  BeamState beam_state(int beam, int bnat) {
    BeamState bs;
    bs.beam = beam;
    bs.bnat = bnat;
    bs.cap = cap_max;
    bs.feed = s_feed;
    bs.score = s_score;
    bs.greedy = b_greedy;
    bs.anchors[0] = s_anchors;
    bs.anchors[1] = b_anchors2;
    bs.hist[0] = s_hist;
    bs.hist[1] = s_hist2;
    bs.live_n = b_live;
    bs.done = s_done;
    bs.nsteps = s_nsteps;
    bs.n_fin = b_nfin;
    bs.greedy_done = b_gdone;
    bs.caps = s_caps;
    bs.f_count = b_fcount;
    bs.f_list = b_flist;
    bs.f_gslot = b_fgslot;
    bs.f_score = b_fscore;
    bs.f_len = b_flen;
    bs.f_forced = b_fforced;
    bs.f_tok = b_ftok;
    bs.E = E;
    bs.pe = pe;
    bs.ln_g = dec[0].ln1g;
    bs.ln_b = dec[0].ln1b;
    bs.x = s1.x;
    bs.y = s1.y;
    bs.scale = emb_scale;
    bs.d = d;
    return bs;
  }

  // Stage-I decoder layers of <= 4 greedy rows on one 16-CTA cluster (decode_cluster.cuh)
  int cluster_decode_mode = 1;  // option "cluster_decode": 1 auto (d 512, ff 2048, 8 heads), 0 off
  int cluster_decode_state = -1;  // -1 unknown, 0 unavailable on this device, 1 available
  int dc_dbg = 0;                 // option "dc_dbg" (timing attribution only)
  bool attn_pdl = true;           // option "attn_pdl" (debug)
  bool cluster_decode_ok(int R) {
    if constexpr (!BF16) return false;
    const int Rp = path_rows > 0 ? path_rows : R;
    // mode 1 (default): single-row buckets, where the cluster kernel measured faster than the
    // per-kernel chain (33.1 vs 34.7 us per batch-1 step); mode 2: buckets up to 4 rows
    const int rmax = cluster_decode_mode >= 2 ? DC_RMAX : 1;
    if (!cluster_decode_mode || d != DC_D || ff != DC_FF || H != DC_H || Ld > DC_MAXL || Rp > rmax || s1_skip ||
        ln_fusable(R))
      return false;
    if (cluster_decode_state < 0) {
      auto prep = [&](auto kern, int smem) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
          return false;
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(DC_CN);
        c.blockDim = dim3(DC_THREADS);
        c.dynamicSmemBytes = smem;
        int n = 0;
        return cudaOccupancyMaxActiveClusters(&n, kern, &c) == cudaSuccess && n >= 1;
      };
      const bool ok = prep(decode_cluster_kernel<1>, DcSmem<1>::TOTAL) &&
                      prep(decode_cluster_kernel<2>, DcSmem<2>::TOTAL) && prep(decode_cluster_kernel<4>, DcSmem<4>::TOTAL);
      cudaGetLastError();
      cluster_decode_state = ok ? 1 : 0;
    }
    return cluster_decode_state == 1;
  }
  void launch_decode_cluster(int R, int t, const int* src_off, const int* src_len, const StepCtl* ctl) {
    DcParams dp{};
    for (int i = 0; i < Ld; ++i) {
      const DecW& w = dec[i];
      auto b = [](const T* q) { return reinterpret_cast<const bf16*>(q); };
      dp.L[i] = DcLayer{b(w.wqkv), b(w.wo), b(w.wqc), b(w.woc), b(w.w1), b(w.w2), w.bqkv, w.bo, w.bqc, w.boc, w.b1,
                        w.b2, w.ln2g, w.ln2b, w.ln3g, w.ln3b, i + 1 < Ld ? dec[i + 1].ln1g : dec_lng,
                        i + 1 < Ld ? dec[i + 1].ln1b : dec_lnb};
    }
    dp.Ld = Ld;
    dp.xkv = reinterpret_cast<const bf16*>(xkv);
    dp.xstride = Ld * 2 * d;
    dp.src_off = src_off;
    dp.src_len = src_len;
    dp.kc = reinterpret_cast<bf16*>(s1.kc);
    dp.vc = reinterpret_cast<bf16*>(s1.vc);
    dp.cap = cap_max;
    dp.rcap = R_max;
    dp.x = s1.x;
    dp.y = reinterpret_cast<bf16*>(s1.y);
    dp.ctl = ctl;
    dp.R_host = R;
    dp.t_host = t;
    dp.att_scale = att_scale;
    dp.dbg = dc_dbg;
    Scope sc(this, K_GEMM | K_ATTN, 2.0 * Ld * (6.0 * d * d + 2.0 * d * ff), 2.0 * R * Ld * (6.0 * d * d + 2.0 * d * ff));
    const int Rp = path_rows > 0 ? path_rows : R;
    if (Rp <= 1)
      launch(decode_cluster_kernel<1>, DC_CN, DC_THREADS, DcSmem<1>::TOTAL, dp);
    else if (Rp <= 2)
      launch(decode_cluster_kernel<2>, DC_CN, DC_THREADS, DcSmem<2>::TOTAL, dp);
    else
      launch(decode_cluster_kernel<4>, DC_CN, DC_THREADS, DcSmem<4>::TOTAL, dp);
    check_launch();
  }

  // One Stage-I step for R live rows (R is an upper bound when ctl != null):
  // decoder layers, vocab statistics, selection (greedy or beam), which also
  // embeds the next step's inputs.
  // fuse_advance (plain loop graphs): a greedy bucket of <= 4 rows selects and advances the
  // control block in one launch (greedy_select_advance_kernel); returns true when it did
  bool sel_adv = true;  // option "sel_adv"
  bool stage1_step(int R, int t, int k, int beam, int max_src, const int* src_off, const int* src_len,
                   const GreedyState& gs, const BeamState& bs, StepCtl* ctl, bool fuse_advance = false) {
    const int* Rd = ctl ? &ctl->R : nullptr;
    if (beam == 1) {
      const bool fuse = ln_fusable(R) && !(s1_skip & 1);  // final LN inside the vocab GEMV
      greedy_hist_identity = true;  // greedy rows never reorder: slot j of row r is row r
      try {
        if (cluster_decode_ok(R)) {
          Tag _tgc(this, "s1.decoder_cluster");
          launch_decode_cluster(R, t, src_off, src_len, ctl);
        } else {
          decoder_step(R, t, t * k, cap_max, s_feed, s_hist, nullptr, src_off, src_len, max_src, ctl, false, nullptr,
                       fuse);
        }
      } catch (...) {
        greedy_hist_identity = false;
        throw;
      }
      greedy_hist_identity = false;
      {
        Tag _tg(this, "s1.vocab");
        if (!(s1_skip & 8)) vocab_parts(s1.y, R_max, R, s1.parts, 1, 0, s1.logits, Rd, fuse ? dec_lng : nullptr);
      }
      Tag _tg(this, "s1.select");
      Scope sc(this, K_OTHER, 0, 0);
      if (fuse_advance && sel_adv && ctl && R <= 4 && !(s1_skip & 16)) {
        launch(greedy_select_advance_kernel<T>, 1, 128, 0, s1.parts, gs, R, ctl, (const int*)s_alive);
        check_launch();
        return true;
      }
      if (!(s1_skip & 16)) {
        launch(greedy_select_kernel<T, 1>, cdiv(R, 4), 128, 0, s1.parts, gs, R, t, k, ctl);
        check_launch();
      }
    } else {
      decoder_step(R, t, t * k, cap_max, s_feed, s_hist, s_rowseq, src_off, src_len, max_src, ctl, false, s_hist2);
      {
        Tag _tg(this, "s1.vocab");
        if (!(s1_skip & 8)) vocab_parts(s1.y, R_max, R, s1.parts, beam + 1, 0, s1.logits, Rd);
      }
      Tag _tg(this, "s1.select");
      Scope sc(this, K_OTHER, 0, 0);
      if (!(s1_skip & 16)) {
        if (beam + 1 <= 5)
          launch(rowstat_kernel<5>, cdiv(R, 4), 128, 0, s1.parts, R, beam + 1, s1.rowstat, Rd);
        else
          launch(rowstat_kernel<KTOP_MAX>, cdiv(R, 4), 128, 0, s1.parts, R, beam + 1, s1.rowstat, Rd);
        check_launch();
      }
      if (!(s1_skip & 32)) {
        const int S = cdiv(R, beam);
        launch(beam_select_kernel<T>, S, 32 * BEAM_MAX, 0, s1.rowstat, bs, S, t, k, ctl);
        check_launch();
      }
    }
    return false;
  }

  // Capture (once per row bucket and beam width) the Stage-I step as the body
  // of a conditional WHILE node. Every step-varying value lives in s_ctl.
  // U consecutive Stage-I steps captured as one plain graph (no conditional
  // node: every kernel boundary inside keeps its programmatic (PDL) edge)
  int graph_unroll = 16;  // option "graph_unroll" (0: conditional WHILE loop graph; measured slower)
  std::map<int, LoopGraph> plain_graphs;
  LoopGraph& plain_graph(int bucket, int beam, int U, const GreedyState& gs, const BeamState& bs) {
    LoopGraph& lg = plain_graphs[((bucket * 16 + beam) * 16 + bs.bnat) * 64 + U];
    if (lg.exec) return lg;
    const int64_t before = stats.kernel_launches;
    CUDA_OK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed));
    try {
      for (int u = 0; u < U; ++u) {
        if (!stage1_step(bucket, 0, 0, beam, Lmax, s_srcoff, s_srclen, gs, bs, s_ctl, true)) {
          launch(stage1_advance_plain_kernel, 1, bucket <= 32 ? 32 : 256, 0, s_ctl, s_alive,
                 beam == 1 ? (const int*)s_done : nullptr);
          check_launch();
        }
      }
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(stream, &dummy);
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(stream, &lg.graph));
    lg.kernels = (int)(stats.kernel_launches - before) / U;
    stats.kernel_launches = before;
    CUDA_OK(cudaGraphInstantiate(&lg.exec, lg.graph, 0));
    return lg;
  }
  // Capture every greedy (beam 1, b_nat 1) Stage-I loop graph for row buckets up to `rows`
  // without running them (option "prepare_graphs" = rows): a server or benchmark calls it at
  // setup, so no translate call ever captures (the kernel parameters are fixed pointers, the
  // same GreedyState / BeamState translate() builds, cross-attention prefetch on as in its loop)
  void prepare_graphs(int rows) {
    if (!(BF16 && use_graphs && timed_class == 0 && graph_unroll > 0) || rows < 1) return;
    GreedyState gs{E, pe, dec[0].ln1g, dec[0].ln1b, s1.x, s1.y, emb_scale, d, s_feed, s_done, s_nsteps, s_forced,
                   s_score, s_anchors, s_caps, cap_max};
    BeamState bs = beam_state(1, 1);
    int top = 1;
    while (top < rows) top <<= 1;
    top = std::min(top, R_max);
    const bool pf = cross_prefetch;
    cross_prefetch = true;
    try {
      for (int b = 1;; b = std::min(2 * b, top)) {
        for (int U = graph_unroll; U >= 1; U >>= 1) plain_graph(b, 1, U, gs, bs);
        if (b == top) break;
      }
    } catch (...) {
      cross_prefetch = pf;
      throw;
    }
    cross_prefetch = pf;
  }
  LoopGraph& loop_graph(int bucket, int beam, const GreedyState& gs, const BeamState& bs) {
    // captured kernel parameters depend on the bucket, beam and b_nat (finished-store layout)
    LoopGraph& lg = loop_graphs[(bucket * 16 + beam) * 16 + bs.bnat];
    if (lg.exec) return lg;
    CUDA_OK(cudaGraphCreate(&lg.graph, 0));
    cudaGraphConditionalHandle h;
    CUDA_OK(cudaGraphConditionalHandleCreate(&h, lg.graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CUDA_OK(cudaGraphAddNode(&node, lg.graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int64_t before = stats.kernel_launches;
    CUDA_OK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
      stage1_step(bucket, 0, 0, beam, Lmax, s_srcoff, s_srclen, gs, bs, s_ctl);
      launch(stage1_advance_kernel, 1, 1, 0, s_ctl, s_alive, h);
      check_launch();
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(stream, &dummy);
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(stream, &body));
    lg.kernels = (int)(stats.kernel_launches - before) + 1;
    stats.kernel_launches = before;
    CUDA_OK(cudaGraphInstantiate(&lg.exec, lg.graph, 0));
    return lg;
  }

  void argmax_logprobs(const int32_t* excl, int n_excl, int32_t* amax, float* lp) override;

  void drop_loop_graphs() {  // options that change kernel choice invalidate the captured loops
    for (auto* m : {&loop_graphs, &plain_graphs}) {
      for (auto& kv : *m) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
      }
      m->clear();
    }
  }
  void set_option(const std::string& name, int value) override {
    if (name == "graphs")
      use_graphs = value != 0;
    else if (name == "tail_ln") {
      use_tail_ln = value != 0;
      drop_loop_graphs();
    } else if (name == "pair") {
      pair_mma = value;
      drop_loop_graphs();
    } else if (name == "attn_head_groups") {
      attn_head_groups = std::max(1, value);
    } else if (name == "fill") {
      fill_pct = std::max(1, std::min(100, value));
      drop_loop_graphs();
    } else if (name == "sel_adv") {
      sel_adv = value != 0;
      drop_loop_graphs();
    } else if (name == "prepare_graphs") {
      prepare_graphs(value);
    } else if (name == "balance") {
      balance = value != 0;
      drop_loop_graphs();
    } else if (name == "sm_cap") {
      sm_cap = std::max(0, value);
      drop_loop_graphs();
    } else if (name == "bn32") {
      bn32_mode = value;
      drop_loop_graphs();
    } else if (name == "splitk") {
      use_splitk = value != 0;
      drop_loop_graphs();
    } else if (name == "enc_skip") {
      enc_skip = value;
    } else if (name == "debug_spin") {
      debug_spin_us = value;
    } else if (name == "graph_unroll") {
      if (value < 0 || value > 32 || (value & (value - 1))) throw HrtError(HRT_ERR_INVALID, "graph_unroll: 0 or a power of two <= 32");
      graph_unroll = value;
    } else if (name == "l2_persist") {
      set_l2_persist(value != 0);
      drop_loop_graphs();
    } else if (name == "cluster") {
      cluster_mode = value != 0;
      drop_loop_graphs();
    } else if (name == "cluster_min_mtiles") {
      if (value < 2) throw HrtError(HRT_ERR_INVALID, "cluster_min_mtiles >= 2");
      cluster_min_mtiles = value;
      drop_loop_graphs();
    }
    else if (name == "attn_heads")
      attn_heads_mode = value;
    else if (name == "attn_rows") {
      attn_rows_mode = value;
      drop_loop_graphs();
    }
    else if (name == "attn_pdl") {
      attn_pdl = value != 0;
      drop_loop_graphs();
    } else if (name == "dc_dbg") {
      dc_dbg = value;
      drop_loop_graphs();
    } else if (name == "cluster_decode") {
      cluster_decode_mode = value;
      drop_loop_graphs();
    } else if (name == "cluster4") {
      cluster4 = value;
      drop_loop_graphs();
    } else if (name == "cluster4_min_mtiles") {
      cluster4_min_mtiles = std::max(1, value);
      drop_loop_graphs();
    } else if (name == "ln_row") {
      ln_row = value;
      drop_loop_graphs();
    } else if (name == "ln_row_min_tiles") {
      ln_row_min_tiles = value;
      drop_loop_graphs();
    } else if (name == "res_red") {
      res_red = value != 0;
      drop_loop_graphs();
    } else if (name == "ln_epi") {
      use_ln_epi = value != 0;
      drop_loop_graphs();
    } else if (name == "gemv_rows") {
      if (value < 0 || value > 1024) throw HrtError(HRT_ERR_INVALID, "gemv_rows: 0 .. 1024");
      gemv_rows = value;
      drop_loop_graphs();
    } else if (name == "ln_fuse" || name == "gemv" || name == "gemv_max_m") {
      if (name == "gemv_max_m") {
        if (value != 32 && value != 64 && value != 128) throw HrtError(HRT_ERR_INVALID, "gemv_max_m: 32, 64 or 128");
        gemv_max_m = value;
      } else {
        (name == "gemv" ? use_gemv : use_ln_fuse) = value != 0;
      }
      drop_loop_graphs();
    }
    else if (name == "s1_skip") {  // debug: skip Stage-I kernel classes (timing attribution only; wrong results)
      s1_skip = value;
      drop_loop_graphs();
    }
    else if (name == "stage1_skip") {
      s1_skip = value;
      drop_loop_graphs();
    }
    else
      throw HrtError(HRT_ERR_INVALID, "unknown option " + name);
  }

  void translate(const int32_t* ids, const int32_t* lens, int B, int k, int b_at, int b_nat, float alpha,
                 const int32_t* caps, const hrt_translate_out* out, int on_device, bool at) override;
};

// ---------------------------------------------------------------------------
// weight conversion kernels
// ---------------------------------------------------------------------------
template <typename T>
__global__ void transpose_convert_kernel(const float* __restrict__ s, int K, int N, T* __restrict__ dst) {
  pdl_enter();
  __shared__ float tile[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? s[(size_t)k * N + n] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) dst[(size_t)n * K + k] = from_f<T>(tile[threadIdx.x][i]);
  }
}

template <typename T>
__global__ void convert_kernel(const float* __restrict__ s, size_t n, T* __restrict__ dst) {
  pdl_enter();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = from_f<T>(s[i]);
}

template <typename T>
void Engine<T>::transpose_convert(const float* s, int K, int N, T* dst) {
  dim3 grid(cdiv(N, 32), cdiv(K, 32));
  launch(transpose_convert_kernel<T>, grid, dim3(32, 8), 0, s, K, N, dst);
  check_launch();
}
template <typename T>
void Engine<T>::convert(const float* s, size_t n, T* dst) {
  launch(convert_kernel<T>, 1024, 256, 0, s, n, dst);
  check_launch();
}

// argmax / renormalised log-prob over non-excluded ids (infer.py:401-418)
__global__ void argmax_lp_kernel(const float* __restrict__ logits, int V, const unsigned char* __restrict__ excl,
                                 int* __restrict__ amax, float* __restrict__ lp) {
  pdl_enter();
  const int row = blockIdx.x;
  const float* l = logits + (size_t)row * V;
  __shared__ float sv[32];
  __shared__ int si[32];
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    if (excl && excl[c]) continue;
    if (better(l[c], c, bv, bi)) {
      bv = l[c];
      bi = c;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    sv[0] = bv;
    si[0] = bi;
  }
  __syncthreads();
  const float m = sv[0];
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x)
    if (!(excl && excl[c])) s += expf(l[c] - m);
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sv[w];
    amax[row] = si[0];
    lp[row] = -logf(t);
  }
}

template <typename T>
void Engine<T>::argmax_logprobs(const int32_t* excl, int n_excl, int32_t* amax, float* lp) {
  if (p_B == 0) throw HrtError(HRT_ERR_INFERENCE, "parallel_logits() must precede argmax_logprobs()");
  const int M2 = p_B * p_T;
  meta_reset();
  size_t cur = meta_hdr;
  unsigned char* d_ex = nullptr;
  if (excl && n_excl > 0) {
    std::vector<unsigned char> m(V, 0);
    for (int i = 0; i < n_excl; ++i) {
      if (excl[i] < 0 || excl[i] >= V) throw HrtError(HRT_ERR_INVALID, "excluded id out of range");
      m[excl[i]] = 1;
    }
    std::vector<int> packed((V + 3) / 4, 0);
    std::memcpy(packed.data(), m.data(), V);
    d_ex = reinterpret_cast<unsigned char*>(meta_put(cur, packed));
  }
  int* d_amax = meta_put(cur, std::vector<int>(M2, 0));
  float* d_lp = reinterpret_cast<float*>(meta_put(cur, std::vector<int>(M2, 0)));
  meta_flush(cur);
  launch(argmax_lp_kernel, M2, 256, 0, p_logits, V, d_ex, d_amax, d_lp);
  check_launch();
  stats.kernel_launches++;
  CUDA_OK(cudaMemcpyAsync(amax, d_amax, M2 * sizeof(int), cudaMemcpyDeviceToHost, stream));
  CUDA_OK(cudaMemcpyAsync(lp, d_lp, M2 * sizeof(float), cudaMemcpyDeviceToHost, stream));
  CUDA_OK(cudaStreamSynchronize(stream));
}

// ---------------------------------------------------------------------------
// fused production path: hrt_translate for a batch (decoding.py:249-302)
// ---------------------------------------------------------------------------
template <typename T>
void Engine<T>::translate(const int32_t* ids, const int32_t* lens, int B, int k, int b_at, int b_nat, float alpha,
                          const int32_t* caps, const hrt_translate_out* out, int on_device, bool at) {
  if (B < 1) throw HrtError(HRT_ERR_INVALID, "batch size out of range");
  if (B > Bmax)  // a phase plan larger than the arena (arena.py:38-42)
    throw HrtError(HRT_ERR_MEMORY, "batch of " + std::to_string(B) + " sentences exceeds the arena's max_sentences " +
                                       std::to_string(Bmax));
  // at: the autoregressive baseline (decoding.py:163-185) on the same captured
  // Stage-I loop -- interval 1 from BOS, no Stage II (greedy only on this face)
  if (at && (k != 1 || b_at != 1 || b_nat != 1))
    throw HrtError(HRT_ERR_INVALID, "the fused AT path is greedy (beam 1); use the session protocol for AT beam search");
  if (!at && (k < 2 || k > cfg.max_chunk)) throw HrtError(HRT_ERR_DECODING, "chunk size k not supported by the engine");
  if (b_nat < 1 || b_at < b_nat) throw HrtError(HRT_ERR_DECODING, "need b_at >= b_nat >= 1");
  if (b_at > beam_max) throw HrtError(HRT_ERR_INVALID, "b_at exceeds engine max_beam");
  if (b_at > BEAM_MAX) throw HrtError(HRT_ERR_INVALID, "b_at > 7 unsupported by the device beam search");
  const int beam = b_at, bn = b_nat;
  const bool greedy_mode = beam == 1;
  // ---- host schedule: truncate (decoding.py:260), caps, sort by cap desc ----
  std::vector<int> raw_off(B + 1, 0), S(B), cap(B);
  for (int i = 0; i < B; ++i) {
    if (lens[i] < 1) throw HrtError(HRT_ERR_INVALID, "empty source");
    raw_off[i + 1] = raw_off[i] + lens[i];
    S[i] = std::min<int>(lens[i], Lmax);
    cap[i] = caps ? caps[i] : (at ? Lmax : cdiv(Lmax, k));  // decoding.py:174 / :202-203
    if (cap[i] < 1) throw HrtError(HRT_ERR_INVALID, "max_steps must be >= 1");
    if (cap[i] + 1 > cap_max || k * cap[i] + 1 > P)
      throw HrtError(HRT_ERR_INVALID, "max_steps exceeds the positional table / cache capacity");
  }
  // host ids: validated here (the reference's np.take raises IndexError) and
  // packed already truncated to max_len, so the capacity check sees the
  // truncated total; device ids keep their raw offsets (the gather kernel
  // truncates, and clamps out-of-range ids to EOS instead of reading past E)
  const bool host_io = on_device != 1;
  std::vector<int> trunc_off;
  if (host_io) {
    trunc_off.assign(B + 1, 0);
    for (int i = 0; i < B; ++i) {
      trunc_off[i + 1] = trunc_off[i] + S[i];
      const int32_t* src = ids + raw_off[i];
      for (int j = 0; j < lens[i]; ++j)
        if (src[j] < 0 || src[j] >= V)
          throw HrtError(HRT_ERR_INVALID, "source token id " + std::to_string(src[j]) + " out of range [0, " +
                                              std::to_string(V) + ")");
    }
    if (trunc_off[B] > Me_max) throw HrtError(HRT_ERR_MEMORY, "source tokens exceed max_src_tokens");
  }
  std::vector<int> perm(B);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return cap[a] > cap[b]; });
  const int C = B * bn;  // Stage-II candidates, c = s * b_nat + i
  std::vector<int> off(B + 1, 0), len(B), capS(B), slot(C), off2(C + 1, 0), moff(C + 1, 0);
  int max_src = 0, max_cap = 0, max_slot = 0;
  for (int i = 0; i < B; ++i) {
    const int p = perm[i];
    len[i] = S[p];
    off[i + 1] = off[i] + S[p];
    capS[i] = cap[p];
    max_src = std::max(max_src, S[p]);
    max_cap = std::max(max_cap, cap[p]);
  }
  for (int c = 0; c < C; ++c) {
    slot[c] = k * capS[c / bn];
    off2[c + 1] = off2[c] + slot[c];
    moff[c + 1] = moff[c] + (slot[c] - slot[c] / k);
    max_slot = std::max(max_slot, slot[c]);
  }
  const int Mtok = off[B];
  if (Mtok > Me_max) throw HrtError(HRT_ERR_MEMORY, "source tokens exceed max_src_tokens");
  const int M2 = off2[C], Mm = moff[C];
  if (M2 > M2_max) throw HrtError(HRT_ERR_MEMORY, "stage-II rows exceed capacity");
  for (int ph = 0; ph < (at ? 2 : 3); ++ph) note_high_water(ph, ArenaDims{Mtok, B * beam, M2, Mm});
  // Stage-I rows alive at step t: beam rows of every sentence whose cap > t
  // (a prefix of the cap-sorted batch)
  std::vector<int> alive(max_cap, 0);
  for (int t = 0, r = B; t < max_cap; ++t) {
    while (r > 0 && capS[r - 1] <= t) --r;
    alive[t] = r * beam;
  }
  // mask-row map for the final Stage-II LayerNorm gather
  std::vector<int> out_row(M2, -1), seqmap(C), cand_beg(B + 1);
  for (int c = 0; c < C; ++c) {
    for (int j = 0; j < slot[c]; ++j)
      if ((j + 1) % k != 0) out_row[off2[c] + j] = moff[c] + j - (j + 1) / k;
    seqmap[c] = c / bn;
  }
  for (int s = 0; s <= B; ++s) cand_beg[s] = s * bn;
  meta_reset();
  size_t cur = meta_hdr;
  int* d_rawoff = meta_put(cur, host_io ? trunc_off : raw_off);
  int* d_perm = meta_put(cur, perm);
  int* d_off = meta_put(cur, off);
  int* d_len = meta_put(cur, len);
  int* d_caps = meta_put(cur, capS);
  int* d_slot = meta_put(cur, slot);
  int* d_off2 = meta_put(cur, off2);
  int* d_moff = meta_put(cur, moff);
  int* d_seqmap = meta_put(cur, seqmap);
  int* d_cbeg = meta_put(cur, cand_beg);
  int* d_qlen2 = meta_put(cur, std::vector<int>(C, 0));
  int* d_outrow = meta_put(cur, out_row);
  const std::vector<int> enc_items = prefill_items(len), s2_items = prefill_items(slot);
  int* d_enc_items = meta_put(cur, enc_items);
  int* d_s2_items = meta_put(cur, s2_items);
  // host source ids (truncated) ride in the same pinned metadata copy (one H2D transfer per call)
  int* d_ids_meta = nullptr;
  const bool ids_in_meta = host_io && cur + trunc_off[B] <= (size_t)meta_cap;
  if (ids_in_meta) {
    for (int i = 0; i < B; ++i) std::memcpy(h_meta + cur + trunc_off[i], ids + raw_off[i], (size_t)S[i] * sizeof(int));
    d_ids_meta = d_meta + cur;
    cur = (cur + trunc_off[B] + 7) & ~size_t(7);
  }
  {  // fixed header: loop control + alive[] + source offsets/lengths
    // (timing attribution with kernels skipped produces garbage that may end rows early: the
    // early exit is disabled then, so every step still runs)
    StepCtl c{0, alive.empty() ? 0 : alive[0], 0, k, max_cap, s1_skip ? (1 << 30) : B, 0,
              alive.empty() ? 0 : alive[0]};
    std::memcpy(h_meta, &c, sizeof(StepCtl));
    int* ha = h_meta + 8;
    for (int t = 0; t <= cap_max; ++t) ha[t] = t < max_cap ? alive[t] : 0;
    int* ho = ha + align_up(cap_max + 1, 8);
    std::copy(off.begin(), off.end(), ho);
    std::fill(ho + B + 1, ho + R_max + 1, off[B]);
    int* hl = ho + align_up(R_max + 1, 8);
    std::copy(len.begin(), len.end(), hl);
    std::fill(hl + B, hl + R_max, 0);
  }
  meta_flush(cur);
  const int* src_ids = ids;
  if (d_ids_meta) {
    src_ids = d_ids_meta;
  } else if (host_io) {  // (unreachable with the metadata sizing; kept for a smaller meta_cap)
    for (int i = 0; i < B; ++i)
      CUDA_OK(cudaMemcpyAsync(d_ids_raw + trunc_off[i], ids + raw_off[i], (size_t)S[i] * sizeof(int),
                              cudaMemcpyHostToDevice, stream));
    src_ids = d_ids_raw;
  }
  {
    Scope sc(this, K_OTHER, 8.0 * Mtok, 0);
    launch(gather_sentences_kernel, B, 128, 0, src_ids, d_rawoff, d_off, d_perm, d_ids, d_pos, B, V);
    check_launch();
  }
  if (debug_spin_us > 0) debug_spin_kernel<<<1, 32, 0, stream>>>((long long)debug_spin_us * 1000);
  // ---- phase 1: encoder ----
  phase_mark(0);
  run_encoder(Mtok, B, max_src, d_off, d_len, d_enc_items, (int)enc_items.size() / 2);
  phase_mark(1);
  // ---- phase 2: Stage I (decoding.py:90-155) ----
  // cache capacity max_steps + 1 (start_cache, decoding.py:97); the fused path
  // keeps the engine-wide stride cap_max so captured graphs stay valid
  const int capA = cap_max;
  const int bos = at ? BOS_ID : 4 + (k - 2);  // BOS / BOS_k (data.py:14-16)
  CUDA_OK(cudaMemcpyAsync(s_caps, d_caps, B * sizeof(int), cudaMemcpyDeviceToDevice, stream));
  GreedyState gs{E, pe, dec[0].ln1g, dec[0].ln1b, s1.x, s1.y, emb_scale, d,
                 s_feed, s_done, s_nsteps, s_forced, s_score, s_anchors, s_caps, capA};
  BeamState bs = beam_state(beam, bn);
  {
    Scope sc(this, K_OTHER, 0, 0);
    if (greedy_mode)
      launch(stage1_init_kernel, cdiv(B, 128), 128, 0, B, capA, bos, s_feed, s_done, s_nsteps, s_forced, s_score,
             s_hist);
    else
      launch(beam_init_kernel, cdiv(B * beam, 128), 128, 0, bs, B, bos);
    check_launch();
    if (!greedy_mode) {
      launch(rowseq_fill_kernel, cdiv(R_max, 128), 128, 0, s_rowseq, B * beam, R_max, beam, B);
      check_launch();
    }
  }
  {  // step-0 input (BOS_k at position 0); later steps are embedded by the selection kernel
    Tag _tg(this, "s1.embed_ln");
    embed_ln(s_feed, nullptr, 0, alive.empty() ? 0 : alive[0], dec[0].ln1g, dec[0].ln1b, s1.x, s1.y);
  }
  // Stage-I steps in segments of constant row bucket (power of two >= live
  // rows): each segment is one launch of its bucket's captured loop graph, so
  // kernel choice and grid size follow the shrinking batch (small buckets take
  // the mma.sync GEMV path)
  auto bucket_of = [&](int r) {
    int b = 1;
    while (b < r) b <<= 1;
    return std::min(b, R_max);
  };
  struct PrefetchScope {  // cross-attention K/V prefetch is valid inside this loop only
    bool& f;
    explicit PrefetchScope(bool& flag) : f(flag) { f = true; }
    ~PrefetchScope() { f = false; }
  } pscope(cross_prefetch);
  unrolled_last = false;
  for (int t0 = 0; t0 < max_cap && alive[t0] > 0;) {
    const int bucket = bucket_of(alive[t0]);
    int t1 = t0;
    while (t1 < max_cap && alive[t1] > 0 && bucket_of(alive[t1]) == bucket) ++t1;
    const bool unrolled = BF16 && use_graphs && timed_class == 0 && graph_unroll > 0;
    unrolled_last = unrolled;
    if (!unrolled || t0 == 0) {
      // loop control (the finished count carries over); the copy also orders every
      // earlier kernel (encoder) before Stage I (cross_prefetch relies on it). The
      // unrolled graphs need it once: their advance kernel steps t / R / pos across
      // segment boundaries, and sets R = 0 once every row has finished (natural EOS,
      // decoding.py:149-150), so the remaining captured steps exit at once.
      const int hdr[5] = {t0, alive[t0], t0 * k, k, unrolled ? max_cap : t1};
      CUDA_OK(cudaMemcpyAsync(s_ctl, hdr, sizeof(hdr), cudaMemcpyHostToDevice, stream));
    }
    if (unrolled) {
      // n steps as U-step graphs, U = graph_unroll, graph_unroll / 2, ..., 1
      // (binary decomposition: at most log2(graph_unroll) + 1 graphs per bucket)
      int left = t1 - t0;
      // capture every size of every bucket up to this call's largest on first use, so a
      // later call whose tail ends in a bucket this one never reached (few long sentences)
      // does not capture inside a timed region
      {
        const int top = bucket_of(alive[0]);
        for (int b = 1;; b = std::min(2 * b, top)) {
          for (int U = graph_unroll; U >= 1; U >>= 1) plain_graph(b, beam, U, gs, bs);
          if (b == top) break;
        }
      }
      for (int U = graph_unroll; U >= 1 && left > 0; U >>= 1) {
        if (left < U) continue;
        LoopGraph& lg = plain_graph(bucket, beam, U, gs, bs);
        while (left >= U) {
          CUDA_OK(cudaGraphLaunch(lg.exec, stream));
          stats.kernel_launches += (int64_t)lg.kernels * U;
          left -= U;
        }
      }
    } else if (BF16 && use_graphs && timed_class == 0) {
      LoopGraph& lg = loop_graph(bucket, beam, gs, bs);
      CUDA_OK(cudaGraphLaunch(lg.exec, stream));
      stats.kernel_launches += (int64_t)lg.kernels * (t1 - t0);
    } else {
      path_rows = bucket;  // same kernel choices as the captured loop
      try {
        for (int t = t0; t < t1; ++t) stage1_step(alive[t], t, k, beam, max_src, d_off, d_len, gs, bs, nullptr);
      } catch (...) {
        path_rows = 0;
        throw;
      }
      path_rows = 0;
    }
    t0 = t1;
  }
  phase_mark(2);
  // ---- phase 3: Stage II over the selected candidates ----
  Stage2Cands cands;
  if (at) {
    cands = Stage2Cands{s_anchors, nullptr, capA, s_nsteps, s_score, s_forced, s_nsteps};
  } else if (greedy_mode) {
    cands = Stage2Cands{s_anchors, nullptr, capA, s_nsteps, s_score, s_forced, s_nsteps};
  } else {
    Scope sc(this, K_OTHER, 0, 0);
    launch(beam_candidates_kernel, cdiv(B, 128), 128, 0, bs, B, c_off, c_len, c_sat, c_forced);
    check_launch();
    cands = Stage2Cands{b_ftok, c_off, capA, c_len, c_sat, c_forced, bs.nsteps};
  }
  if (!at) {
    {
      Scope sc(this, K_OTHER, 0, 0);
      launch(stage2_build_kernel, C, 128, 0, cands, d_off2, d_slot, C, k, s2.ids, s2.pos, d_qlen2);
      check_launch();
    }
    decoder_parallel(M2, C, max_slot, max_src, d_off2, d_slot, d_qlen2, d_seqmap, d_off, d_len, nullptr, 0, d_outrow,
                     d_s2_items, (int)s2_items.size() / 2);
    Tag _tg2(this, "stage2.vocab");
    vocab_parts(s2.ymask, Mm_max, Mm, s2.parts, 1, 1, s2.logits);
    {
      Scope sc(this, K_OTHER, 0, 0);
      launch(rowstat_kernel<1>, cdiv(Mm, 4), 128, 0, s2.parts, Mm, 1, s2.mstat, (const int*)nullptr);
      check_launch();
    }
  }
  Stage2Out so;
  so.tokens = host_io ? o_tokens : out->tokens;
  so.lens = host_io ? o_lens : out->lens;
  so.scores = host_io ? o_scores : out->scores;
  so.calls = host_io ? o_calls : out->calls;
  so.forced = host_io ? o_forced : out->forced;
  // synchronous host I/O: the five outputs of this call are packed back to back
  // (sized by B, inside the o_* region) so one D2H copy returns them all
  const size_t pk_len = (size_t)B * Lmax * sizeof(int), pk_calls = pk_len + B * sizeof(int),
               pk_scores = align_up(pk_calls + B * sizeof(int), 8), pk_forced = pk_scores + (size_t)B * 3 * sizeof(double),
               pk_total = pk_forced + B;
  const bool packed = host_io && on_device == 0 && h_out != nullptr && pk_total <= h_out_bytes;
  if (packed) {
    char* pb = reinterpret_cast<char*>(o_tokens);
    so.tokens = reinterpret_cast<int*>(pb);
    so.lens = reinterpret_cast<int*>(pb + pk_len);
    so.calls = reinterpret_cast<int*>(pb + pk_calls);
    so.scores = reinterpret_cast<double*>(pb + pk_scores);
    so.forced = reinterpret_cast<unsigned char*>(pb + pk_forced);
  }
  so.out_index = d_perm;
  {
    Scope sc(this, K_OTHER, 0, 0);
    if (at)
      launch(at_finish_kernel, cdiv(B, 4), 128, 0, cands, alpha, Lmax, B, so);
    else
      launch(stage2_finish_kernel, cdiv(B, 4), 128, 0, s2.ids, d_off2, d_qlen2, d_moff, s2.mstat, d_cbeg, cands, k,
             alpha, Lmax, B, so);
    check_launch();
  }
  phase_mark(3);
  phase_valid = true;
  // rows the Stage-I loop computed (device row counts, unrolled-graph path): statistics
  const bool row_stat = unrolled_last && host_io && on_device == 0;
  if (row_stat) CUDA_OK(cudaMemcpyAsync(h_ctl, s_ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost, stream));
  if (packed) {
    CUDA_OK(cudaMemcpyAsync(h_out, o_tokens, pk_total, cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaStreamSynchronize(stream));
    std::memcpy(out->tokens, h_out, pk_len);
    std::memcpy(out->lens, h_out + pk_len, B * sizeof(int));
    std::memcpy(out->calls, h_out + pk_calls, B * sizeof(int));
    std::memcpy(out->scores, h_out + pk_scores, (size_t)B * 3 * sizeof(double));
    std::memcpy(out->forced, h_out + pk_forced, B);
    for (int i = 0; i < B; ++i) stats.decoder_calls += out->calls[i];
    if (row_stat) stats.stage1_row_steps += h_ctl->pad;
  } else if (host_io) {
    CUDA_OK(cudaMemcpyAsync(out->tokens, o_tokens, (size_t)B * Lmax * sizeof(int), cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaMemcpyAsync(out->lens, o_lens, B * sizeof(int), cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaMemcpyAsync(out->scores, o_scores, B * 3 * sizeof(double), cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaMemcpyAsync(out->calls, o_calls, B * sizeof(int), cudaMemcpyDeviceToHost, stream));
    CUDA_OK(cudaMemcpyAsync(out->forced, o_forced, B, cudaMemcpyDeviceToHost, stream));
    if (on_device == 0) {  // 2: host buffers, caller synchronises (concurrent engines)
      CUDA_OK(cudaStreamSynchronize(stream));
      for (int i = 0; i < B; ++i) stats.decoder_calls += out->calls[i];
      if (row_stat) stats.stage1_row_steps += h_ctl->pad;
    }
  }
}

}  // namespace hrt
