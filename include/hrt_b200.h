/*
 * hrt_b200.h — C ABI of the B200-native Hybrid-Regressive Translation engine.
 *
 * The reference (arXiv 2212.01543 desk-scale package, /root/reference/pkg/src/hrt)
 * exposes this path as a Python session object driven by decoding.py. This
 * header is the drop-in boundary that replaces it: plain pointers and sizes,
 * no framework types. Two faces:
 *
 *   1. session protocol (step-level parity with the reference):
 *        hrt_encode            <- InferenceSession.encode          infer.py:176-221
 *        hrt_start_cache       <- InferenceSession.start_cache     infer.py:225-232
 *        hrt_step              <- InferenceSession.step            infer.py:234-305
 *        hrt_reorder           <- InferenceSession.reorder         infer.py:307-318
 *        hrt_parallel_logits   <- InferenceSession.parallel_logits infer.py:322-399
 *        hrt_argmax_logprobs   <- InferenceSession.argmax_logprobs infer.py:401-418
 *   2. fused production call:
 *        hrt_translate_batch   <- decoding.hrt_translate, batched  decoding.py:249-302
 *                                 (encoder -> Stage-I skip-AT -> Stage-II fill -> selection)
 *
 * Ownership: the caller owns every host buffer passed in or out; the engine
 * owns weights, its activation arena and KV caches. One engine serves one
 * device and one host thread; calls are serialised on the engine's stream.
 * Every call returns an hrt_status; hrt_last_error() gives the message.
 * Status codes map to the reference's exceptions in the Python wrapper:
 *   HRT_ERR_INVALID   -> ValueError / ModelError      (model.py:21)
 *   HRT_ERR_INFERENCE -> InferenceError               (infer.py:23)
 *   HRT_ERR_DECODING  -> DecodingError                (decoding.py:31)
 *   HRT_ERR_MEMORY    -> ArenaOverflowError           (arena.py:15)
 */
#ifndef HRT_B200_H
#define HRT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HRT_OK = 0,
  HRT_ERR_INVALID = 1,
  HRT_ERR_INFERENCE = 2,
  HRT_ERR_DECODING = 3,
  HRT_ERR_MEMORY = 4,
  HRT_ERR_CUDA = 5
} hrt_status;

enum { HRT_DTYPE_F32 = 0, HRT_DTYPE_BF16 = 1 };

/* Model shape (ModelConfig, model.py:25-62) plus engine capacity. */
typedef struct hrt_config {
  int32_t d_model, d_ff, n_heads, enc_layers, dec_layers, vocab_size, max_len;
  int32_t max_chunk;      /* largest supported k; PE rows = max_len + max_chunk + 1 */
  int32_t dtype;          /* HRT_DTYPE_F32 | HRT_DTYPE_BF16 (bf16 weights/activations, fp32 accumulate) */
  int32_t max_sentences;  /* sentences per hrt_translate_batch / hrt_encode call */
  int32_t max_beam;       /* largest b_at */
  int32_t max_src_tokens; /* packed source tokens per call; 0 -> max_sentences * max_len */
} hrt_config;

typedef struct hrt_engine hrt_engine;

typedef struct hrt_stats {
  int64_t kernel_launches;   /* kernels this engine launched (all calls) */
  int64_t decoder_calls;     /* reference decoder-call counter (infer.py:161) */
  int64_t arena_bytes;       /* device activation arena capacity (hrt_estimate_arena max) */
  int64_t arena_high_water;  /* largest phase footprint any call needed (<= arena_bytes) */
  int64_t weight_bytes;      /* device weight blob */
  int64_t stage1_row_steps;  /* Stage-I rows computed, summed over steps (captured-graph loop, host I/O
                                calls): below sum(cap) once rows stop at a natural EOS */
} hrt_stats;

/* Create an engine on `device`. `params` holds every parameter as fp32, in
 * the reference's insertion order (model.py:146-181: embed, enc.{i}.{ln1,attn,
 * ln2,ffn}, enc.final_ln, dec.{i}.{ln1,attn,ln2,cross,ln3,ffn}, dec.final_ln),
 * matrices row-major (d_in, d_out). n_params must equal hrt_param_count(cfg). */
hrt_status hrt_create(const hrt_config* cfg, const float* params, int64_t n_params, int32_t device,
                      hrt_engine** out);
void hrt_destroy(hrt_engine* eng);
int64_t hrt_param_count(const hrt_config* cfg);
const char* hrt_last_error(const hrt_engine* eng);  /* eng may be NULL: last global error */
/* Closed-form activation-arena bytes per phase for an engine of this config
 * (estimate_max_bytes, infer.py:78-96): phase_bytes[0] encoder, [1] skip-AT
 * (Stage I), [2] skip-CMLM (Stage II), [3] max = the arena capacity that
 * hrt_create allocates. Phases alias one allocation. No GPU needed. */
hrt_status hrt_estimate_arena(const hrt_config* cfg, int64_t* phase_bytes);
hrt_status hrt_get_stats(const hrt_engine* eng, hrt_stats* out);
void* hrt_stream(hrt_engine* eng);                  /* the engine's cudaStream_t */
hrt_status hrt_synchronize(hrt_engine* eng);

/* ---- session protocol --------------------------------------------------- */
/* Encode n_seq sources (packed ids, lens[i] tokens each). memory_out (host,
 * nullable) receives the final-LN'd encoder output, sum(lens) x d_model fp32. */
hrt_status hrt_encode(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t n_seq, float* memory_out);
/* Start a causal decode of `rows` rows with `cap` cached steps; row_seq (host,
 * nullable) names the encoded sequence each row attends (default 0). */
hrt_status hrt_start_cache(hrt_engine* eng, int32_t rows, int32_t cap, const int32_t* row_seq);
/* One decoder call at `position` for every row; logp_out (host, nullable)
 * receives rows x vocab fp32 full-vocabulary log-probs. */
hrt_status hrt_step(hrt_engine* eng, const int32_t* tokens, int32_t position, float* logp_out);
/* Row j continues from old row parents[j]. */
hrt_status hrt_reorder(hrt_engine* eng, const int32_t* parents);
/* One parallel decoder pass over B x T inputs; mode 0 = full, 1 = causal;
 * pad_mask (nullable) nonzero where the input is a real token; seq (nullable)
 * names the encoded sequence per row of the batch. logits_out (nullable)
 * receives B x T x vocab fp32; the logits stay on device for argmax_logprobs. */
hrt_status hrt_parallel_logits(hrt_engine* eng, const int32_t* ids, const int32_t* positions, const uint8_t* pad_mask,
                               int32_t B, int32_t T, int32_t mode, const int32_t* seq, float* logits_out);
/* Per-position argmax over the non-excluded ids and its log-softmax value
 * renormalised over them, for the last parallel_logits call. */
hrt_status hrt_argmax_logprobs(hrt_engine* eng, const int32_t* exclude, int32_t n_exclude, int32_t* amax_out,
                               float* lp_out);

/* ---- fused production call ---------------------------------------------- */
typedef struct hrt_translate_out {
  int32_t* tokens;   /* [B][max_len]; row i holds lens[i] tokens */
  int32_t* lens;     /* [B] */
  double* scores;    /* [B][3] = skip_at_score, skip_cmlm_score, score */
  int32_t* calls;    /* [B] decoder_calls = Stage-I steps + 1 */
  uint8_t* forced;   /* [B] finished by the Stage-I cap */
} hrt_translate_out;

/* Translate B sentences. ids: packed source tokens (sum(lens) entries);
 * sources longer than max_len keep their first max_len tokens (decoding.py:260);
 * host ids outside [0, vocab_size) fail with HRT_ERR_INVALID (np.take's
 * IndexError), device-resident ids (io_on_device 1) are clamped to EOS;
 * lens and max_steps are HOST arrays (the schedule); max_steps NULL means the
 * reference default ceil(max_len / k) (decoding.py:202-203). When
 * io_on_device is 0, ids and every output pointer are host memory and the
 * copies are part of the call; when 1 they are device memory; when 2 they are
 * (pinned) host memory and the call returns without synchronising -- the
 * caller uses hrt_synchronize (concurrent engines on one device). */
hrt_status hrt_translate_batch(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t B, int32_t k,
                               int32_t b_at, int32_t b_nat, float length_penalty, const int32_t* max_steps,
                               const hrt_translate_out* out, int32_t io_on_device);

/* Autoregressive baseline (decoding.at_translate, decoding.py:163-185) on the
 * same kernels and captured Stage-I loop: interval 1 from BOS, no Stage II.
 * Greedy only (beam must be 1; AT beam search runs through the session
 * protocol). max_steps NULL means max_len steps. Outputs as for
 * hrt_translate_batch: scores = {s, 0, s / len^length_penalty}, calls = steps. */
hrt_status hrt_at_translate_batch(hrt_engine* eng, const int32_t* ids, const int32_t* lens, int32_t B, int32_t beam,
                                  float length_penalty, const int32_t* max_steps, const hrt_translate_out* out,
                                  int32_t io_on_device);

/* Engine options (speed only; "graphs", "graph_unroll", "cluster", "cluster4" are bit-identical, the kernel-path
 * switches change the bf16 summation order):
 *   "graphs"        1 (default): Stage-I steps replayed from captured CUDA graphs; 0: launched step by step
 *   "graph_unroll"  steps per captured graph (power of two <= 32, default 16); 0: one conditional
 *                   WHILE-node graph per row bucket (the original design, measured slower)
 *   "cluster"       1 (default): large-M tcgen05 GEMMs as CTA pairs sharing the weight tile
 *   "cluster4"      0 (default); 1: clusters of four CTAs sharing it, from "cluster4_min_mtiles"
 *                   row tiles up (same bits; measured slower)
 *   "ln_row"        1 (default, d = 512, bf16): residual projection + following LayerNorm in one
 *                   launch (cta_group::2 CTA pairs, whole 512-column rows per CTA, TMA-staged
 *                   epilogue); 0: GEMM + LayerNorm kernel; 2 / 3: register-epilogue variants
 *   "res_red"       1 (default): residual GEMM epilogues as L2 reductions (same bits)
 *   "balance"       1 (default): persistent GEMM grids sized to the rounds they need (same bits)
 *   "sel_adv"       1 (default): greedy buckets of <= 4 rows select and advance in one launch
 *   "prepare_graphs" n: capture every greedy Stage-I loop graph for up to n rows now (setup call
 *                   for servers / benchmarks, so no later call captures)
 *   "fill", "bn32", "attn_rows": tile width / decode-attention choices; fill=20, bn32=0,
 *                   attn_rows=2 is the throughput mode for several engines sharing one GPU
 *   "gemv", "gemv_max_m", "attn_heads", "splitk", "ln_fuse", "tail_ln", "sm_cap",
 *   "l2_persist": kernel-path switches documented in DESIGN.md §4 / §7. */
hrt_status hrt_set_option(hrt_engine* eng, const char* name, int32_t value);

/* ---- measurement helpers ------------------------------------------------ */
/* Kernel-class timing: when enabled, CUDA events bracket every launch of the
 * named class ("vocab", "gemm", "attn", "all") on the engine stream. */
hrt_status hrt_timing_enable(hrt_engine* eng, const char* kernel_class, int32_t enable);
/* Device milliseconds of the last hrt_translate_batch's phases:
 * ms3[0] encoder (+cross-K/V), ms3[1] Stage I loop, ms3[2] Stage II + selection. */
hrt_status hrt_phase_times(hrt_engine* eng, float* ms3);
/* JSON {"call-site tag": [device ms, launches], ...} of the timed launches since enable. */
hrt_status hrt_timing_report(hrt_engine* eng, char* buf, int64_t cap);
/* Total device milliseconds and launch count of the timed class since enable. */
hrt_status hrt_timing_read(hrt_engine* eng, double* total_ms, int64_t* launches, double* alg_bytes,
                           double* alg_flops);

#ifdef __cplusplus
}
#endif
#endif /* HRT_B200_H */
