// Non-GEMM kernels of the HRT inference path (sm_100a).
//
// Every kernel cites the reference operation it implements
// (/root/reference/pkg/src/hrt/...). Residual streams are fp32; matrix
// operands (T) are fp32 or bf16; all reductions accumulate in fp32, and
// search scores in fp64 as the reference's Python floats do.
#pragma once
#include "common.cuh"

namespace hrt {

constexpr int KTOP_MAX = 8;  // top-k width kept per vocab row (beam <= 7)

// ---------------------------------------------------------------------------
// embedding (+ positional) fused with the first LayerNorm
//   x = E[id] * sqrt(d) + PE[pos]            infer.py:187-189, :250-252, :344-347
//   y = LN(x)                                kernels.py:42-57 (pop. variance, eps 1e-5)
// one warp per row; NPL = ceil(d / 32) values per lane kept in registers.
// ---------------------------------------------------------------------------
template <typename T, int NPL>
__global__ void embed_ln_kernel(const int* __restrict__ ids, const int* __restrict__ pos, int pos_const,
                                const int* __restrict__ M_dev, int M, int d, float scale, const T* __restrict__ E,
                                const float* __restrict__ pe, const float* __restrict__ g,
                                const float* __restrict__ b, float* __restrict__ x, T* __restrict__ y) {
  if (M_dev) M = *M_dev;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int id = ids[row];
  const int p = pos ? pos[row] : pos_const;
  float v[NPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      v[i] = __fadd_rn(__fmul_rn(to_f(E[(size_t)id * d + j]), scale), pe[(size_t)p * d + j]);
      s += v[i];
    } else {
      v[i] = 0.f;
    }
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      const float c = v[i] - mean;
      q += c * c;
    }
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      x[(size_t)row * d + j] = v[i];
      y[(size_t)row * d + j] = from_f<T>((v[i] - mean) * inv * g[j] + b[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// LayerNorm of the fp32 residual stream (kernels.py:42-57). Optional row map:
// out_row[r] >= 0 writes row r to that output row, < 0 skips it (used to
// gather only Stage-II [MASK] rows into the vocab GEMM operand).
// ---------------------------------------------------------------------------
template <typename T, int NPL>
__global__ void layernorm_kernel(const float* __restrict__ x, const int* __restrict__ M_dev, int M, int d,
                                 const float* __restrict__ g, const float* __restrict__ b, T* __restrict__ y,
                                 const int* __restrict__ out_row, float* __restrict__ y32) {
  if (M_dev) M = *M_dev;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int orow = out_row ? out_row[row] : row;
  if (orow < 0) return;
  float v[NPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < d ? x[(size_t)row * d + j] : 0.f;
    s += v[i];
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      const float c = v[i] - mean;
      q += c * c;
    }
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      const float o = (v[i] - mean) * inv * g[j] + b[j];
      y[(size_t)orow * d + j] = from_f<T>(o);
      if (y32) y32[(size_t)orow * d + j] = o;
    }
  }
}

// ---------------------------------------------------------------------------
// Ragged ("varlen") multi-head attention for whole sequences:
//   encoder self-attention            infer.py:196-203   (full)
//   Stage-II self-attention           infer.py:364-373   (full or causal, key padding)
//   Stage-II cross-attention          infer.py:377-385   (keys = sentence memory)
// Sequence s owns query rows [q_off[s], q_off[s] + q_slot[s]) of which the
// first q_len[s] are real (the rest get zero output), and attends key rows
// [kv_off[kvs], kv_off[kvs] + kv_len[kvs]) with kvs = kv_map ? kv_map[s] : s.
// Keys whose key_ok byte is 0 are masked (additive -1e9 in the reference).
// grid = (n_seq, heads, query chunks); one warp per query row; K^T and V of
// the (sequence, head) live in shared memory as fp32.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) attn_prefill_kernel(
    const T* __restrict__ q, int q_stride, const T* __restrict__ k, const T* __restrict__ v, int kv_stride,
    T* __restrict__ out, int out_stride, const int* __restrict__ q_off, const int* __restrict__ q_slot,
    const int* __restrict__ q_len, const int* __restrict__ kv_map, const int* __restrict__ kv_off,
    const int* __restrict__ kv_len, const unsigned char* __restrict__ key_ok, int causal, int dh, int lk_max,
    float scale) {
  extern __shared__ float sm[];
  const int s = blockIdx.x, h = blockIdx.y;
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qslot = q_slot[s];
  const int qbeg = blockIdx.z * nwarp * 8;
  if (qbeg >= qslot) return;
  const int qend = min(qslot, qbeg + nwarp * 8);
  const int qlen = q_len[s];
  const int kvs = kv_map ? kv_map[s] : s;
  const int kb = kv_off[kvs];
  const int L = kv_len[kvs];
  float* Kt = sm;                       // [dh][lk_max]
  float* Vs = Kt + dh * lk_max;         // [lk_max][dh]
  float* kbias = Vs + lk_max * dh;      // [lk_max]
  float* wsc = kbias + lk_max;          // [nwarp][lk_max]
  float* wq = wsc + nwarp * lk_max;     // [nwarp][dh]
  const int hoff = h * dh;
  for (int idx = threadIdx.x; idx < L * dh; idx += blockDim.x) {
    const int j = idx / dh, c = idx - j * dh;
    const size_t r = (size_t)(kb + j) * kv_stride + hoff + c;
    Kt[c * lk_max + j] = to_f(k[r]);
    Vs[j * dh + c] = to_f(v[r]);
  }
  for (int j = threadIdx.x; j < L; j += blockDim.x)
    kbias[j] = (key_ok == nullptr || key_ok[kb + j]) ? 0.f : -INFINITY;
  __syncthreads();
  float* sc = wsc + warp * lk_max;
  float* qv = wq + warp * dh;
  const int qb = q_off[s];
  for (int i = qbeg + warp; i < qend; i += nwarp) {
    T* o = out + (size_t)(qb + i) * out_stride + hoff;
    if (i >= qlen) {
      for (int c = lane; c < dh; c += 32) o[c] = from_f<T>(0.f);
      continue;
    }
    const T* qr = q + (size_t)(qb + i) * q_stride + hoff;
    for (int c = lane; c < dh; c += 32) qv[c] = to_f(qr[c]);
    __syncwarp();
    const int jend = causal ? min(L, i + 1) : L;
    float mx = -INFINITY;
    for (int j = lane; j < jend; j += 32) {
      float a = 0.f;
      for (int c = 0; c < dh; ++c) a = fmaf(qv[c], Kt[c * lk_max + j], a);
      a = a * scale + kbias[j];
      sc[j] = a;
      mx = fmaxf(mx, a);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < jend; j += 32) {
      const float e = (sc[j] == -INFINITY) ? 0.f : __expf(sc[j] - mx);
      sc[j] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    __syncwarp();
    const float inv = sum > 0.f ? 1.0f / sum : 0.f;
    for (int c = lane; c < dh; c += 32) {
      float a = 0.f;
      for (int j = 0; j < jend; ++j) a = fmaf(sc[j], Vs[j * dh + c], a);
      o[c] = from_f<T>(a * inv);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Single-query attention for one Stage-I decoder step (infer.py:259-285).
// SELF: append this step's k/v at cache slot t, then attend slots 0..t of the
//       row's history; history slot j of logical row r lives in physical row
//       hist[r * cap + j] (beam reorder = index permutation, infer.py:307-318).
// CROSS: attend the row's sentence memory keys (computed once in encode).
// One warp per (row, head).
// ---------------------------------------------------------------------------
template <typename T, bool SELF>
__global__ void __launch_bounds__(128) attn_decode_kernel(
    const T* __restrict__ q, int q_stride, const T* __restrict__ knew, const T* __restrict__ vnew, int new_stride,
    T* __restrict__ kc, T* __restrict__ vc, int c_stride, const int* __restrict__ hist, int cap, int t,
    const int* __restrict__ row_seq, const int* __restrict__ kv_off, const int* __restrict__ kv_len,
    const int* __restrict__ R_dev, int R, int heads, int dh, int lk_max, float scale, T* __restrict__ out,
    int out_stride) {
  extern __shared__ float sm[];
  if (R_dev) R = *R_dev;
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * nwarp + warp;
  if (item >= R * heads) return;
  const int r = item / heads, h = item - r * heads;
  float* sc = sm + warp * (lk_max + dh);
  float* qv = sc + lk_max;
  const int hoff = h * dh;
  for (int c = lane; c < dh; c += 32) qv[c] = to_f(q[(size_t)r * q_stride + hoff + c]);
  int L;
  const T* kbase;
  const T* vbase;
  size_t kv_row0 = 0;
  if (SELF) {
    L = t + 1;
    // append this step's key/value (infer.py:259-260)
    const size_t dst = ((size_t)r * cap + t) * c_stride + hoff;
    for (int c = lane; c < dh; c += 32) {
      kc[dst + c] = knew[(size_t)r * new_stride + hoff + c];
      vc[dst + c] = vnew[(size_t)r * new_stride + hoff + c];
    }
    kbase = kc;
    vbase = vc;
  } else {
    const int sq = row_seq ? row_seq[r] : r;
    L = kv_len[sq];
    kv_row0 = kv_off[sq];
    kbase = knew;
    vbase = vnew;
  }
  __syncwarp();
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) {
    const T* kr;
    if (SELF) {
      kr = (j == t) ? knew + (size_t)r * new_stride + hoff
                    : kbase + ((size_t)hist[(size_t)r * cap + j] * cap + j) * c_stride + hoff;
    } else {
      kr = kbase + (kv_row0 + j) * (size_t)new_stride + hoff;
    }
    float a = 0.f;
    for (int c = 0; c < dh; ++c) a = fmaf(qv[c], to_f(kr[c]), a);
    a *= scale;
    sc[j] = a;
    mx = fmaxf(mx, a);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < L; j += 32) {
    const float e = __expf(sc[j] - mx);
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.0f / sum;
  for (int c = lane; c < dh; c += 32) {
    float a = 0.f;
    for (int j = 0; j < L; ++j) {
      const T* vr;
      if (SELF) {
        vr = (j == t) ? vnew + (size_t)r * new_stride + hoff
                      : vbase + ((size_t)hist[(size_t)r * cap + j] * cap + j) * c_stride + hoff;
      } else {
        vr = vbase + (kv_row0 + j) * (size_t)new_stride + hoff;
      }
      a = fmaf(sc[j], to_f(vr[c]), a);
    }
    out[(size_t)r * out_stride + hoff + c] = from_f<T>(a * inv);
  }
}

// ---------------------------------------------------------------------------
// Vocabulary statistics.
// The vocab projection (infer.py:293-301 Stage I; :395-396 + :409-418 Stage II)
// never materialises log-probs on the production path: each N-tile of the
// logits GEMM emits per-row partials {max, sum exp(l - max), top-k allowed},
// and a per-row merge produces the final normaliser and top-k.
//   norm_allowed = 0 : normaliser over the full vocabulary (Stage I)
//   norm_allowed = 1 : normaliser over the generable set  (Stage II, argmax_logprobs)
// ---------------------------------------------------------------------------
struct VocabParts {
  float* mx;   // [rows][ntiles]
  float* sum;  // [rows][ntiles]
  float* val;  // [rows][ntiles][KT]
  int* id;     // [rows][ntiles][KT]
  float* eos;  // [rows]   logit of EOS (tile 0 owns column 2)
  int ntiles;
};

struct RowStat {
  float mx;    // normaliser max
  float lse;   // log sum exp(l - mx)
  float eos;   // logit of EOS
  int kt;
  float val[KTOP_MAX];
  int id[KTOP_MAX];
};

// Per-thread running accumulator over a contiguous run of columns of one row.
template <int KT>
struct TileAcc {
  float mx, sum;
  float val[KT];
  int id[KT];
  __device__ __forceinline__ void init() {
    mx = -INFINITY;
    sum = 0.f;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      val[i] = -INFINITY;
      id[i] = 0x7fffffff;
    }
  }
  __device__ __forceinline__ void insert(float v, int c) {
    if (!better(v, c, val[KT - 1], id[KT - 1])) return;
    int p = KT - 1;
#pragma unroll
    for (int i = KT - 1; i > 0; --i) {
      if (p == i && better(v, c, val[i - 1], id[i - 1])) {
        val[i] = val[i - 1];
        id[i] = id[i - 1];
        p = i - 1;
      }
    }
    val[p] = v;
    id[p] = c;
  }
  // columns col0 .. col0+n-1 with logits l[0..n)
  __device__ __forceinline__ void add(const float* l, int col0, int n, int norm_allowed) {
    float cm = -INFINITY;
    for (int i = 0; i < n; ++i) {
      const int c = col0 + i;
      const bool ok = id_allowed(c);
      if (!norm_allowed || ok) cm = fmaxf(cm, l[i]);
      if (ok) insert(l[i], c);
    }
    if (cm == -INFINITY) return;
    if (cm > mx) {
      sum *= __expf(mx - cm);
      mx = cm;
    }
    for (int i = 0; i < n; ++i) {
      const int c = col0 + i;
      if (!norm_allowed || id_allowed(c)) sum += __expf(l[i] - mx);
    }
  }
};

// tcgen05 epilogue: one thread owns one row of a 128 x BN logits tile.
template <int KT>
struct VocabEpi {
  VocabParts parts;
  int norm_allowed;
  int bn;
  struct State {
    TileAcc<KT> acc;
  };
  __device__ __forceinline__ void begin(State& s, int, int) const { s.acc.init(); }
  __device__ __forceinline__ void chunk(State& s, int row, int col0, const float* v, int n) const {
    if (col0 <= EOS_ID && EOS_ID < col0 + n) parts.eos[row] = v[EOS_ID - col0];
    s.acc.add(v, col0, n, norm_allowed);
  }
  __device__ __forceinline__ void end(State& s, int row, int n0) const {
    const int tile = n0 / bn;
    const size_t o = (size_t)row * parts.ntiles + tile;
    parts.mx[o] = s.acc.mx;
    parts.sum[o] = s.acc.sum;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      parts.val[o * KT + i] = s.acc.val[i];
      parts.id[o * KT + i] = s.acc.id[i];
    }
  }
};

// Same partials from a materialised fp32 logits matrix (fp32 SIMT path and
// parity/debug mode). grid = (rows, ntiles), one warp per (row, 256-col tile):
// each lane accumulates a strided subset, then lanes merge.
template <int KT>
__global__ void rowstats_from_logits_kernel(const float* __restrict__ logits, int ld, int V,
                                            const int* __restrict__ row_map, VocabParts parts, int tile_w,
                                            int norm_allowed) {
  const int row = blockIdx.x, tile = blockIdx.y, lane = threadIdx.x;
  const int src = row_map ? row_map[row] : row;
  const float* l = logits + (size_t)src * ld;
  const int c0 = tile * tile_w, c1 = min(V, c0 + tile_w);
  TileAcc<KT> a;
  a.init();
  for (int c = c0 + lane; c < c1; c += 32) {
    float x = l[c];
    a.add(&x, c, 1, norm_allowed);
    if (c == EOS_ID) parts.eos[row] = x;
  }
  // merge lanes: max + rescaled sum
  const float m = warp_max(a.mx);
  float s = (a.mx == -INFINITY) ? 0.f : a.sum * __expf(a.mx - m);
  s = warp_sum(s);
  // top-k merge: KT rounds of warp arg-best over each lane's head
  float hv[KT];
  int hid[KT];
  int head = 0;
  for (int r = 0; r < KT; ++r) {
    float v = head < KT ? a.val[head] : -INFINITY;
    int id = head < KT ? a.id[head] : 0x7fffffff;
    float bv = v;
    int bid = id;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
      if (better(ov, oid, bv, bid)) {
        bv = ov;
        bid = oid;
      }
    }
    hv[r] = bv;
    hid[r] = bid;
    if (head < KT && id == bid && bid != 0x7fffffff) ++head;
  }
  if (lane == 0) {
    const size_t o = (size_t)row * parts.ntiles + tile;
    parts.mx[o] = m;
    parts.sum[o] = s;
    for (int i = 0; i < KT; ++i) {
      parts.val[o * KT + i] = hv[i];
      parts.id[o * KT + i] = hid[i];
    }
  }
}

// Warp-level merge of a row's tile partials into a RowStat (lane 0 returns it).
template <int KT>
__device__ __forceinline__ RowStat merge_row(const VocabParts& parts, int row, int kt) {
  const int lane = threadIdx.x & 31;
  const size_t base = (size_t)row * parts.ntiles;
  float m = -INFINITY;
  for (int t = lane; t < parts.ntiles; t += 32) m = fmaxf(m, parts.mx[base + t]);
  m = warp_max(m);
  float s = 0.f;
  for (int t = lane; t < parts.ntiles; t += 32) {
    const float tm = parts.mx[base + t];
    if (tm != -INFINITY) s += parts.sum[base + t] * __expf(tm - m);
  }
  s = warp_sum(s);
  RowStat rs;
  rs.mx = m;
  rs.lse = logf(s);
  rs.eos = parts.eos[row];
  rs.kt = kt;
  // kt <= KT rounds; in round r every lane scans its tiles' sorted lists for
  // the best entry strictly worse than the previous round's winner.
  float pv = INFINITY;
  int pid = -1;
  for (int r = 0; r < kt; ++r) {
    float bv = -INFINITY;
    int bid = 0x7fffffff;
    for (int t = lane; t < parts.ntiles; t += 32) {
      for (int i = 0; i < KT; ++i) {
        const float v = parts.val[(base + t) * KT + i];
        const int id = parts.id[(base + t) * KT + i];
        if (id == 0x7fffffff) break;
        if (better(pv, pid, v, id) && better(v, id, bv, bid)) {
          bv = v;
          bid = id;
          break;  // lists are sorted: first entry worse than the previous winner is this tile's best
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oid = __shfl_xor_sync(0xffffffffu, bid, o);
      if (better(ov, oid, bv, bid)) {
        bv = ov;
        bid = oid;
      }
    }
    rs.val[r] = bv;
    rs.id[r] = bid;
    pv = bv;
    pid = bid;
  }
  return rs;
}

// ---------------------------------------------------------------------------
// Stage-I greedy selection (decoding.py:102-150 with beam = 1): one warp per
// live row merges its vocab partials; lane 0 applies the reference rules.
//   token  = EOS at the sentence's last allowed step (forced), else the
//            lowest-id argmax over the generable set;
//   score += fp32 log-softmax value of the token (full-vocab normaliser),
//            accumulated in fp64.
// ---------------------------------------------------------------------------
struct GreedyState {
  int* feed;       // [rows] next fed token
  int* done;       // [rows]
  int* nsteps;     // [rows] steps taken when finished
  int* forced;     // [rows]
  double* score;   // [rows]
  int* anchors;    // [rows][cap]
  const int* caps; // [rows] Stage-I step cap (max_steps)
  int cap;
};

template <int KT>
__global__ void greedy_select_kernel(VocabParts parts, GreedyState st, int R, int t) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= R) return;
  if (st.done[row]) return;
  const RowStat rs = merge_row<KT>(parts, row, 1);
  if (lane != 0) return;
  const bool last = (t == st.caps[row] - 1);
  const int tok = last ? EOS_ID : rs.id[0];
  const float logit = last ? rs.eos : rs.val[0];
  const float lp = (logit - rs.mx) - rs.lse;
  st.score[row] += (double)lp;
  st.anchors[(size_t)row * st.cap + t] = tok;
  st.feed[row] = tok;
  if (tok == EOS_ID) {
    st.done[row] = 1;
    st.nsteps[row] = t + 1;
    st.forced[row] = last ? 1 : 0;
  }
}

// Final per-row stats (protocol face / Stage II): amax + renormalised logprob.
template <int KT>
__global__ void rowstat_kernel(VocabParts parts, int R, int kt, RowStat* __restrict__ out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= R) return;
  const RowStat rs = merge_row<KT>(parts, row, kt);
  if ((threadIdx.x & 31) == 0) out[row] = rs;
}

// ---------------------------------------------------------------------------
// Stage-II input (decoding.py:208-217, :268-276): candidate c (sentence
// cand_sent[c]) with m anchors gets slot rows [off[c], off[c] + slot[c]):
// position j < k*m holds MASK, or the anchor z_{(j+1)/k-1} when (j+1) % k == 0;
// positions are j + 1. Rows past k*m are padding (never attended, ignored).
// ---------------------------------------------------------------------------
__global__ void stage2_build_kernel(const int* __restrict__ anchors, int cap, const int* __restrict__ cand_row,
                                    const int* __restrict__ cand_len, const int* __restrict__ off,
                                    const int* __restrict__ slot, int C, int k, int* __restrict__ ids,
                                    int* __restrict__ pos, int* __restrict__ qlen) {
  const int c = blockIdx.x;
  if (c >= C) return;
  const int m = cand_len[c];
  const int T = k * m;
  const int sl = slot[c], o = off[c];
  const int* z = anchors + (size_t)cand_row[c] * cap;
  if (threadIdx.x == 0) qlen[c] = T;
  for (int j = threadIdx.x; j < sl; j += blockDim.x) {
    int id = PAD_ID;
    if (j < T) id = ((j + 1) % k == 0) ? z[(j + 1) / k - 1] : MASK_ID;
    ids[o + j] = id;
    pos[o + j] = j + 1;
  }
}

// ---------------------------------------------------------------------------
// Stage-II fill, Eq.(2) score and output (decoding.py:280-302).
// One warp per sentence; candidates cand_beg[s] .. cand_beg[s+1]-1.
//   filled_j  = amax_j at MASK positions, anchors pass through
//   s_cmlm    = sum of renormalised logprobs at MASK positions (fp64)
//   score     = (s_at + s_cmlm) / (k*m)^alpha ; best = first strict maximum
//   tokens    = truncate(truncate_at_eos(filled), max_len)
// mask_row[c][j] indexes the vocab-stat row of MASK position j (slot layout).
// ---------------------------------------------------------------------------
struct Stage2Out {
  int* tokens;       // [S][max_len]
  int* lens;         // [S]
  double* scores;    // [S][3] = skip_at, skip_cmlm, score
  int* calls;        // [S]
  unsigned char* forced;  // [S]
  const int* out_index;   // [S] -> output slot (undo the length sort)
};

__global__ void stage2_finish_kernel(const int* __restrict__ ids, const int* __restrict__ off,
                                     const int* __restrict__ qlen, const int* __restrict__ mrow_off,
                                     const RowStat* __restrict__ mstat, const int* __restrict__ cand_beg,
                                     const int* __restrict__ cand_row, const double* __restrict__ s_at,
                                     const int* __restrict__ nsteps, const int* __restrict__ forced, int k,
                                     float alpha, int max_len, int S, Stage2Out out) {
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  int best = -1;
  double best_score = 0.0, best_cmlm = 0.0;
  for (int c = cand_beg[s]; c < cand_beg[s + 1]; ++c) {
    const int T = qlen[c];
    const int o = off[c];
    double part = 0.0;
    // MASK positions j (in slot layout) map to consecutive stat rows
    const int mo = mrow_off[c];
    for (int j = lane; j < T; j += 32) {
      if ((j + 1) % k != 0) {
        const int mi = j - (j + 1) / k;  // index among this candidate's MASK rows
        const RowStat& rs = mstat[mo + mi];
        part += (double)(-rs.lse);
      }
    }
    (void)o;
    const double cmlm = warp_sum_d(part);
    const double sc = (s_at[cand_row[c]] + cmlm) / pow((double)T, (double)alpha);
    if (best < 0 || sc > best_score) {
      best = c;
      best_score = sc;
      best_cmlm = cmlm;
    }
  }
  const int c = best;
  const int T = qlen[c];
  const int o = off[c];
  const int mo = mrow_off[c];
  const int dst = out.out_index ? out.out_index[s] : s;
  // first EOS in the filled sequence (warp scan over positions)
  int first_eos = T;
  for (int j0 = 0; j0 < T; j0 += 32) {
    const int j = j0 + lane;
    int tok = -1;
    if (j < T) {
      tok = ((j + 1) % k != 0) ? mstat[mo + j - (j + 1) / k].id[0] : ids[o + j];
    }
    const unsigned ball = __ballot_sync(0xffffffffu, j < T && tok == EOS_ID);
    if (ball) {
      first_eos = j0 + __ffs(ball) - 1;
      break;
    }
  }
  const int n = min(first_eos, max_len);
  for (int j = lane; j < n; j += 32) {
    const int tok = ((j + 1) % k != 0) ? mstat[mo + j - (j + 1) / k].id[0] : ids[o + j];
    out.tokens[(size_t)dst * max_len + j] = tok;
  }
  if (lane == 0) {
    const int r = cand_row[c];
    out.lens[dst] = n;
    out.scores[(size_t)dst * 3 + 0] = s_at[r];
    out.scores[(size_t)dst * 3 + 1] = best_cmlm;
    out.scores[(size_t)dst * 3 + 2] = best_score;
    out.calls[dst] = nsteps[r] + 1;
    out.forced[dst] = (unsigned char)forced[r];
  }
}

// ---------------------------------------------------------------------------
// small utility kernels
// ---------------------------------------------------------------------------
// packed gather of sentences into a new order: dst sentence i <- src sentence perm[i]
__global__ void gather_sentences_kernel(const int* __restrict__ src, const int* __restrict__ src_off,
                                        const int* __restrict__ dst_off, const int* __restrict__ perm,
                                        int* __restrict__ dst, int* __restrict__ pos, int n) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int p = perm[i];
  const int so = src_off[p], len = src_off[p + 1] - so, d0 = dst_off[i];
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    dst[d0 + j] = src[so + j];
    pos[d0 + j] = j;
  }
}

// Stage-I row initialisation: feed = bos, history slot map = identity.
__global__ void stage1_init_kernel(int R, int cap, int bos, int* feed, int* done, int* nsteps, int* forced,
                                   double* score, int* hist) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  feed[r] = bos;
  done[r] = 0;
  nsteps[r] = 0;
  forced[r] = 0;
  score[r] = 0.0;
  for (int j = 0; j < cap; ++j) hist[(size_t)r * cap + j] = r;
}

// Beam reorder as an index permutation (infer.py:307-318): row j continues
// from old row parents[j]; history slots 0..t-1 follow the parent.
__global__ void reorder_hist_kernel(const int* __restrict__ parents, const int* __restrict__ hist_in,
                                    int* __restrict__ hist_out, int R, int cap, int t) {
  const int r = blockIdx.x;
  if (r >= R) return;
  const int p = parents[r];
  for (int j = threadIdx.x; j < cap; j += blockDim.x)
    hist_out[(size_t)r * cap + j] = (j < t) ? hist_in[(size_t)p * cap + j] : r;
}

// Full-row log-softmax in place (protocol-face step(), infer.py:296-301).
__global__ void logsoftmax_rows_kernel(float* __restrict__ l, int ld, int V) {
  const int row = blockIdx.x;
  float* x = l + (size_t)row * ld;
  __shared__ float red[32];
  float m = -INFINITY;
  for (int c = threadIdx.x; c < V; c += blockDim.x) m = fmaxf(m, x[c]);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    v = warp_max(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) s += expf(x[c] - m);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float lse = logf(red[0]);
  for (int c = threadIdx.x; c < V; c += blockDim.x) x[c] = (x[c] - m) - lse;
}

// fp32 -> bf16 conversion (weights, once at engine creation)
__global__ void f32_to_bf16_kernel(const float* __restrict__ a, bf16* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __float2bfloat16_rn(a[i]);
}

}  // namespace hrt
