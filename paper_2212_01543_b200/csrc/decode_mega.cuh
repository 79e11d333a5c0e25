// Stage-I tail megakernel: when at most MG_RMAX rows are still decoding,
// per-step work is a handful of GEMVs whose cost is pure kernel latency on
// the regular path (~14 launches per step). This cooperative persistent
// kernel runs ALL remaining greedy Stage-I steps (decoding.py:102-150 with
// beam = 1) in one launch: one CTA per SM, phases separated by grid barriers,
// LayerNorms folded into the prologue of the phase that consumes them.
//
//   per step, per decoder layer (infer.py:253-292):
//     [LN1]QKV (+ K/V append) | self-attn | Wo (+res) | [LN2]Qc | cross-attn |
//     Woc (+res) | [LN3]W1 (ReLU) | W2 (+res)
//   then [final LN]vocab statistics (infer.py:293-301) | selection + next
//   step's embedding (same rules as greedy_select_kernel).
//
// GEMV phases: warp w of the grid takes output features n = w, w + W, ...;
// the 32 lanes split K into 16-byte bf16 vectors, activations (<= 8 rows) sit
// in shared memory as fp32, and each feature's dot products are warp-reduced.
// Weights stream from L2/HBM once per step.
#pragma once
#include "kernels.cuh"

namespace hrt {

constexpr int MG_RMAX = 8;
constexpr int MG_THREADS = 512;
constexpr int MG_WARPS = MG_THREADS / 32;
constexpr int MG_MAX_LAYERS = 4;

struct MegaLayer {
  const bf16 *wqkv, *wo, *wqc, *woc, *w1, *w2;
  const float *bqkv, *bo, *bqc, *boc, *b1, *b2, *ln1g, *ln1b, *ln2g, *ln2b, *ln3g, *ln3b;
};

struct MegaParams {
  int d, ff, H, V, Ld, cap, k, rcap;
  MegaLayer L[MG_MAX_LAYERS];
  const float *lng, *lnb;
  const bf16* E;
  const float* pe;
  float scale, att_scale;
  const bf16* xkv;
  int xstride;
  const int *src_off, *src_len;
  bf16 *kc, *vc;  // [Ld][rcap][cap][d]
  float* x;       // [rows][d] residual stream (shared with the regular path)
  float *qkv, *ctx, *hid, *vpart, *veos;
  GreedyState st;
  StepCtl* ctl;
  const int* alive;
  unsigned* bar;  // [2]: arrival count, generation
  int t_begin, t_end, nrows;
  unsigned long long* trace;  // optional: globaltimer at each barrier of the first step (block 0)
};

__device__ __forceinline__ unsigned long long mg_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void mg_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

// rows [0, R) of src (ld K) into shared memory; optional LayerNorm (one warp per row)
__device__ __forceinline__ void mg_stage_rows(const float* src, int R, int K, const float* g, const float* b,
                                              float* sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += MG_WARPS) {
    const float* xr = src + (size_t)r * K;
    float* o = sm + (size_t)r * K;
    if (g == nullptr) {
      for (int j = lane * 4; j < K; j += 128) *reinterpret_cast<float4*>(o + j) = __ldcg(reinterpret_cast<const float4*>(xr + j));
      continue;
    }
    float s = 0.f;
    for (int j = lane * 4; j < K; j += 128) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(xr + j));
      *reinterpret_cast<float4*>(o + j) = v;
      s += (v.x + v.y) + (v.z + v.w);
    }
    const float mean = warp_sum(s) / K;
    float q = 0.f;
    for (int j = lane * 4; j < K; j += 128) {
      const float4 v = *reinterpret_cast<const float4*>(o + j);
      q += (v.x - mean) * (v.x - mean) + (v.y - mean) * (v.y - mean) + (v.z - mean) * (v.z - mean) +
           (v.w - mean) * (v.w - mean);
    }
    const float inv = 1.0f / sqrtf(warp_sum(q) / K + 1e-5f);
    for (int j = lane * 4; j < K; j += 128) {
      float4 v = *reinterpret_cast<const float4*>(o + j);
      v.x = (v.x - mean) * inv * g[j] + b[j];
      v.y = (v.y - mean) * inv * g[j + 1] + b[j + 1];
      v.z = (v.z - mean) * inv * g[j + 2] + b[j + 2];
      v.w = (v.w - mean) * inv * g[j + 3] + b[j + 3];
      *reinterpret_cast<float4*>(o + j) = v;
    }
  }
  __syncthreads();
}

// dot products of NF consecutive-stride weight rows (bf16, K) with the R
// staged rows; all NF x K/256 vector loads are issued before the math so a
// warp keeps several L2/HBM requests in flight; every lane returns all
// results (warp-reduced). acc[f][r].
template <int NF>
__device__ __forceinline__ void mg_dotn(const bf16* const* w, const float* sm, int R, int K, float (*acc)[MG_RMAX]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int r = 0; r < MG_RMAX; ++r) acc[f][r] = 0.f;
  for (int k0 = lane * 8; k0 < K; k0 += 256) {
    float wv[NF][8];
#pragma unroll
    for (int f = 0; f < NF; ++f) load8(w[f] + k0, wv[f]);
#pragma unroll
    for (int r = 0; r < MG_RMAX; ++r) {
      if (r < R) {
        const float4 a = *reinterpret_cast<const float4*>(sm + (size_t)r * K + k0);
        const float4 bq = *reinterpret_cast<const float4*>(sm + (size_t)r * K + k0 + 4);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          float s = acc[f][r];
          s = fmaf(wv[f][0], a.x, s);
          s = fmaf(wv[f][1], a.y, s);
          s = fmaf(wv[f][2], a.z, s);
          s = fmaf(wv[f][3], a.w, s);
          s = fmaf(wv[f][4], bq.x, s);
          s = fmaf(wv[f][5], bq.y, s);
          s = fmaf(wv[f][6], bq.z, s);
          s = fmaf(wv[f][7], bq.w, s);
          acc[f][r] = s;
        }
      }
    }
  }
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int r = 0; r < MG_RMAX; ++r)
      if (r < R) acc[f][r] = warp_sum(acc[f][r]);
}

__device__ __forceinline__ void mg_dot(const bf16* w, const float* sm, int R, int K, float* acc) {
  float a[1][MG_RMAX];
  const bf16* wp[1] = {w};
  mg_dotn<1>(wp, sm, R, K, a);
#pragma unroll
  for (int r = 0; r < MG_RMAX; ++r) acc[r] = a[0][r];
}

// GEMV phase driver: features n = gw + j*GW, processed 4 at a time; fn(n, acc[R]) per feature
template <class Fn>
__device__ __forceinline__ void mg_gemv(const bf16* W, int N, int K, const float* sm, int R, int gw, int GW, Fn fn) {
  int n = gw;
  for (; n + 3 * GW < N; n += 4 * GW) {
    const bf16* w[4] = {W + (size_t)n * K, W + (size_t)(n + GW) * K, W + (size_t)(n + 2 * GW) * K,
                        W + (size_t)(n + 3 * GW) * K};
    float acc[4][MG_RMAX];
    mg_dotn<4>(w, sm, R, K, acc);
#pragma unroll
    for (int f = 0; f < 4; ++f) fn(n + f * GW, acc[f]);
  }
  for (; n < N; n += GW) {
    float acc[MG_RMAX];
    mg_dot(W + (size_t)n * K, sm, R, K, acc);
    fn(n, acc);
  }
}

// one decode-attention item (row r, head h), dh = 64 (infer.py:259-285)
template <bool SELF>
__device__ __forceinline__ void mg_attention(const MegaParams& p, int layer, int r, int h, int t, float* sc) {
  constexpr int DH = 64;
  const int lane = threadIdx.x & 31;
  const int d = p.d;
  const float* qsrc = SELF ? p.qkv + (size_t)r * 3 * d : p.qkv + (size_t)r * 3 * d;  // Q (self) / Qc (cross) in cols [0,d)
  float qr[DH];
#pragma unroll
  for (int c = 0; c < DH; c += 4) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(qsrc + h * DH + c));
    qr[c] = v.x * p.att_scale;
    qr[c + 1] = v.y * p.att_scale;
    qr[c + 2] = v.z * p.att_scale;
    qr[c + 3] = v.w * p.att_scale;
  }
  const size_t lstride = (size_t)p.rcap * p.cap * d;
  const bf16* kbase;
  const bf16* vbase;
  size_t row_stride;
  int L;
  if (SELF) {
    kbase = p.kc + layer * lstride + (size_t)r * p.cap * d + h * DH;
    vbase = p.vc + layer * lstride + (size_t)r * p.cap * d + h * DH;
    row_stride = d;
    L = t + 1;
  } else {
    const size_t o = (size_t)p.src_off[r] * p.xstride + (size_t)2 * layer * d + h * DH;
    kbase = p.xkv + o;
    vbase = p.xkv + o + d;
    row_stride = p.xstride;
    L = p.src_len[r];
  }
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) {
    const bf16* kr = kbase + (size_t)j * row_stride;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int c = 0; c < DH; c += 8) {
      float kk[8];
      load8(kr + c, kk);
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        a0 = fmaf(qr[c + e], kk[e], a0);
        a1 = fmaf(qr[c + e + 1], kk[e + 1], a1);
      }
    }
    sc[j] = a0 + a1;
    mx = fmaxf(mx, a0 + a1);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  for (int j = lane; j < L; j += 32) {
    const float e = ex2f((sc[j] - mx) * LOG2E);
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.0f / sum;
  // PV: 4 groups of 8 lanes, a lane owns 8 head dims
  const int grp = lane >> 3, li = lane & 7;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int j = grp; j < L; j += 4) {
    const float pj = sc[j];
    float vv[8];
    load8(vbase + (size_t)j * row_stride + li * 8, vv);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = fmaf(pj, vv[e], acc[e]);
  }
#pragma unroll
  for (int o = 8; o < 32; o <<= 1)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (grp == 0) {
    float* dst = p.ctx + (size_t)r * d + h * DH + li * 8;
    *reinterpret_cast<float4*>(dst) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(MG_THREADS, 1) decode_mega_kernel(MegaParams p) {
  extern __shared__ float msm[];
  int tr_i = 0;
  auto trace = [&](int t) {
    if (p.trace && t == p.t_begin && blockIdx.x == 0 && threadIdx.x == 0 && tr_i < 63) p.trace[tr_i++] = mg_clock();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * MG_WARPS + warp, GW = gridDim.x * MG_WARPS;
  const int d = p.d, ff = p.ff, H = p.H;
  float* rows = msm;                                                 // MG_RMAX * max(d, ff) staged rows
  float* scw = rows + (size_t)MG_RMAX * (ff > d ? ff : d) + warp * (p.cap + 4);  // per-warp scores
  float* wpart = rows + (size_t)MG_RMAX * (ff > d ? ff : d) + MG_WARPS * (p.cap + 4);  // [warps][R][4]
  for (int t = p.t_begin; t < p.t_end; ++t) {
    const int R = p.alive[t];
    if (R <= 0) break;
    if (*(volatile int*)&p.ctl->finished >= p.nrows) break;
    trace(t);
    for (int i = 0; i < p.Ld; ++i) {
      const MegaLayer& W = p.L[i];
      // ---- [LN1] QKV; append K/V at slot t ----
      mg_stage_rows(p.x, R, d, W.ln1g, W.ln1b, rows);
      mg_gemv(W.wqkv, 3 * d, d, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) {
          const float v = acc[lane] + W.bqkv[n];
          p.qkv[(size_t)lane * 3 * d + n] = v;
          if (n >= d) {
            bf16* cache = (n < 2 * d ? p.kc : p.vc) + (size_t)i * p.rcap * p.cap * d;
            cache[((size_t)lane * p.cap + t) * d + (n - (n < 2 * d ? d : 2 * d))] = __float2bfloat16_rn(v);
          }
        }
      });
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- self attention ----
      for (int it = gw; it < R * H; it += GW) mg_attention<true>(p, i, it / H, it % H, t, scw);
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- Wo + residual ----
      mg_stage_rows(p.ctx, R, d, nullptr, nullptr, rows);
      mg_gemv(W.wo, d, d, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) p.x[(size_t)lane * d + n] = __ldcg(p.x + (size_t)lane * d + n) + (acc[lane] + W.bo[n]);
      });
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- [LN2] Qc ----
      mg_stage_rows(p.x, R, d, W.ln2g, W.ln2b, rows);
      mg_gemv(W.wqc, d, d, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) p.qkv[(size_t)lane * 3 * d + n] = acc[lane] + W.bqc[n];
      });
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- cross attention ----
      for (int it = gw; it < R * H; it += GW) mg_attention<false>(p, i, it / H, it % H, t, scw);
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- Woc + residual ----
      mg_stage_rows(p.ctx, R, d, nullptr, nullptr, rows);
      mg_gemv(W.woc, d, d, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) p.x[(size_t)lane * d + n] = __ldcg(p.x + (size_t)lane * d + n) + (acc[lane] + W.boc[n]);
      });
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- [LN3] W1 + ReLU ----
      mg_stage_rows(p.x, R, d, W.ln3g, W.ln3b, rows);
      mg_gemv(W.w1, ff, d, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) p.hid[(size_t)lane * ff + n] = fmaxf(acc[lane] + W.b1[n], 0.f);
      });
      mg_grid_barrier(p.bar);
      trace(t);
      // ---- W2 + residual ----
      mg_stage_rows(p.hid, R, ff, nullptr, nullptr, rows);
      mg_gemv(W.w2, d, ff, rows, R, gw, GW, [&](int n, const float* acc) {
        if (lane < R) p.x[(size_t)lane * d + n] = __ldcg(p.x + (size_t)lane * d + n) + (acc[lane] + W.b2[n]);
      });
      mg_grid_barrier(p.bar);
      trace(t);
    }
    // ---- [final LN] vocabulary statistics: full-vocab normaliser, top-1 over the generable set ----
    mg_stage_rows(p.x, R, d, p.lng, p.lnb, rows);
    {
      float mx = -INFINITY, sum = 0.f, bv = -INFINITY;
      int bi = 0x7fffffff;
      mg_gemv(p.E, p.V, d, rows, R, gw, GW, [&](int v, const float* acc) {
        if (lane < R) {
          const float l = acc[lane];
          if (v == EOS_ID) p.veos[lane] = l;
          if (l > mx) {
            sum = sum * ex2f((mx - l) * LOG2E) + 1.f;
            mx = l;
          } else {
            sum += ex2f((l - mx) * LOG2E);
          }
          if (id_allowed(v) && better(l, v, bv, bi)) {
            bv = l;
            bi = v;
          }
        }
      });
      if (lane < R) {
        float* wp = wpart + ((size_t)warp * MG_RMAX + lane) * 4;
        wp[0] = mx;
        wp[1] = sum;
        wp[2] = bv;
        wp[3] = __int_as_float(bi);
      }
      __syncthreads();
      if (warp == 0 && lane < R) {  // CTA partial for row `lane`
        float m = -INFINITY;
        for (int w = 0; w < MG_WARPS; ++w) m = fmaxf(m, wpart[((size_t)w * MG_RMAX + lane) * 4]);
        float s = 0.f, cbv = -INFINITY;
        int cbi = 0x7fffffff;
        for (int w = 0; w < MG_WARPS; ++w) {
          const float* wp = wpart + ((size_t)w * MG_RMAX + lane) * 4;
          if (wp[0] != -INFINITY) s += wp[1] * ex2f((wp[0] - m) * LOG2E);
          const int id = __float_as_int(wp[3]);
          if (better(wp[2], id, cbv, cbi)) {
            cbv = wp[2];
            cbi = id;
          }
        }
        float* vp = p.vpart + ((size_t)lane * gridDim.x + blockIdx.x) * 4;
        vp[0] = m;
        vp[1] = s;
        vp[2] = cbv;
        vp[3] = __int_as_float(cbi);
      }
    }
    mg_grid_barrier(p.bar);
      trace(t);
    // ---- selection (block r handles row r) + next step's embedding ----
    if (blockIdx.x < R && warp == 0) {
      const int r = blockIdx.x;
      const GreedyState& st = p.st;
      float m = -INFINITY;
      for (int b = lane; b < gridDim.x; b += 32) m = fmaxf(m, __ldcg(p.vpart + ((size_t)r * gridDim.x + b) * 4));
      m = warp_max(m);
      float s = 0.f, bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int b = lane; b < gridDim.x; b += 32) {
        const float4 vp = __ldcg(reinterpret_cast<const float4*>(p.vpart + ((size_t)r * gridDim.x + b) * 4));
        if (vp.x != -INFINITY) s += vp.y * ex2f((vp.x - m) * LOG2E);
        const int id = __float_as_int(vp.w);
        if (better(vp.z, id, bv, bi)) {
          bv = vp.z;
          bi = id;
        }
      }
      s = warp_sum(s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ov, oi, bv, bi)) {
          bv = ov;
          bi = oi;
        }
      }
      int tok = st.feed[r];
      if (!st.done[r]) {
        if (lane == 0) {
          const bool last = (t == st.caps[r] - 1);
          if (bi == 0x7fffffff) {
            bi = EOS_ID;
            bv = __ldcg(p.veos + r);
          }
          tok = last ? EOS_ID : bi;
          const float logit = last ? __ldcg(p.veos + r) : bv;
          const float lp = (logit - m) - logf(s);
          st.score[r] += (double)lp;
          st.anchors[(size_t)r * st.cap + t] = tok;
          st.feed[r] = tok;
          if (tok == EOS_ID) {
            st.done[r] = 1;
            st.nsteps[r] = t + 1;
            st.forced[r] = last ? 1 : 0;
            atomicAdd(&p.ctl->finished, 1);
          }
        }
        tok = __shfl_sync(0xffffffffu, tok, 0);
      }
      // x = E[tok] * sqrt(d) + PE[(t + 1) k]
      const int pos = (t + 1) * p.k;
      for (int j = lane * 8; j < d; j += 256) {
        float e8[8];
        load8(p.E + (size_t)tok * d + j, e8);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          p.x[(size_t)r * d + j + e] = __fadd_rn(__fmul_rn(e8[e], p.scale), p.pe[(size_t)pos * d + j + e]);
      }
    }
    mg_grid_barrier(p.bar);
      trace(t);
  }
}

}  // namespace hrt
