// Persistent Stage-I decode kernel for small live-row counts (R <= MG_RMAX).
//
// At small R a Stage-I step (decoding.py:102-150 with beam = 1, one
// InferenceSession.step, infer.py:234-305) is a chain of dependent GEMVs and
// attentions whose cost on the regular path is kernel latency, not bytes.
// This kernel runs ALL remaining greedy steps in ONE cooperative launch: one
// CTA per SM, phases separated by a monotonic-counter grid barrier.
//
//   per step, per decoder layer (infer.py:253-292):
//     A [select(t-1) + embed] [LN1] QKV (+K/V append) | B self-attn |
//     C Wo (+res) | D [LN2] Qc | E cross-attn | F Woc (+res) | G [LN3] W1 |
//     H W2 (+res)
//   then I [final LN] vocab statistics (infer.py:293-301).
// The selection of step t-1 (greedy_select_kernel rules) is folded into
// phase A of step t: every CTA that needs a row's next input merges that
// row's vocab partials itself (identical, deterministic result everywhere),
// embeds the chosen token and LayerNorms it; CTA r alone writes row r's
// decoding state. This saves one grid barrier per step.
//
// Projections run on the tensor cores (mma.sync m16n8k16, bf16 in / fp32
// accumulate) with swap-AB: a 16-feature weight tile is the MMA M side and
// the live rows (8 per n-tile) the N side. The K index is permuted
// identically on both operands (lane (g, t) holds k = 8t..8t+7 of each
// 32-wide chunk), so every weight fragment is one 16-byte load. One warp owns
// a tile over (up to) 16 K-chunks, so the epilogue runs from registers; only
// K > 512 splits a tile over several warps of one CTA. Weights do not depend
// on the data: each warp's fragments for the next phase are prefetched with
// cp.async into its shared-memory slot between arriving at and leaving the
// grid barrier, so the copy overlaps the barrier. Attention gives each
// (row, head) a group of 8 warps (32 keys per warp, online-softmax merge).
//
// Numerics mirror the regular path: LN outputs, q/k/v, ctx and the FFN hidden
// layer are rounded to bf16 (the GEMM operand type); the residual stream and
// all accumulations are fp32; scores accumulate in fp64.
#pragma once
#include "kernels.cuh"

namespace hrt {

constexpr int MG_RMAX = 16;  // live rows handled (2 n-tiles of 8)
constexpr int MG_THREADS = 512;
constexpr int MG_WARPS = MG_THREADS / 32;
constexpr int MG_MAX_LAYERS = 4;
constexpr int MG_APAD = 32;   // activation row padding (bf16 elements): conflict-free 16 B fragment loads
constexpr int MG_CPW = 4;     // max K-chunks (32 wide) per warp per tile: a tile's K is split over warps
constexpr int MG_AWARPS = 8;  // warps per attention item (32 keys each per round)

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
  bf16 *q, *ctx, *hid;  // [MG_RMAX][d], [MG_RMAX][d], [MG_RMAX][ff]
  float4* vpart;        // [MG_RMAX][gridDim.x] per-CTA vocab partials {max, sum, best value, best id}
  float* veos;          // [MG_RMAX] logit of EOS
  GreedyState st;
  StepCtl* ctl;
  const int* alive;
  unsigned* bar;  // monotonic arrival counter (zeroed before the launch)
  int t_begin, t_end, nrows;
  int npf;        // prefetch slot capacity per warp, in 32-wide K chunks
  unsigned long long* trace;  // optional: globaltimer at each barrier of step trace_step (block 0)
  int trace_step;
  int skip;  // debug (timing attribution only, results meaningless): bit i skips phase i (A..I = 0..8)
};

__device__ __forceinline__ unsigned long long mg_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier on a monotonic counter, split so work can run between
// arriving (release-add) and waiting (acquire spin): the weight prefetch of
// the next phase overlaps the barrier.
__device__ __forceinline__ void mg_arrive(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void mg_wait(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while ((int)(cur - target) < 0);
  }
  __syncthreads();
}

__device__ __forceinline__ void mg_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// weight fragment load: read-only, no L1 allocation (keeps L1 for the small constants)
__device__ __forceinline__ uint4 ldw16(const bf16* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Work split of a projection (N outputs, K inputs): 16-feature tiles; each
// tile is owned by kspl warps of one CTA (K chunks split evenly, <= 16 each).
// Tile of (CTA c, warp group gi, round q): c + G * (gi + GPC * q).
// ---------------------------------------------------------------------------
struct MgSplit {
  int kspl, cpw, gpc, ntiles;
  __device__ __forceinline__ MgSplit(int N, int K) {
    const int nch = K / 32;
    kspl = 1;
    while (nch / kspl > MG_CPW || nch % kspl) kspl <<= 1;  // host checks K / 32 splits evenly
    cpw = nch / kspl;
    gpc = MG_WARPS / kspl;
    ntiles = (N + 15) / 16;
  }
  __device__ __forceinline__ int rounds() const {
    const int per = gridDim.x * gpc;
    return (ntiles + per - 1) / per;
  }
  __device__ __forceinline__ int tile(int q) const {
    return blockIdx.x + gridDim.x * ((threadIdx.x >> 5) / kspl + gpc * q);
  }
  __device__ __forceinline__ int kpart() const { return (threadIdx.x >> 5) % kspl; }
  // does this CTA own any tile (warp group 0, round 0)?
  __device__ __forceinline__ bool cta_has_work() const { return (int)blockIdx.x < ntiles; }
};

// cp.async this lane's first min(nch, npf) weight chunks of a tile into the
// warp's prefetch slot: pf[(2c) * 32 + lane] = W[n0+g][k0+32c+8t..+8],
// pf[(2c+1) * 32 + lane] = W[n0+g+8][...].
__device__ __forceinline__ void mg_fetch(const bf16* __restrict__ W, int K, int n0, int nvalid, int k0, int nch,
                                         uint4* pf, int npf) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const bf16* w0 = W + (size_t)(n0 + min(g, nvalid - 1)) * K + k0 + t4 * 8;
  const bf16* w1 = W + (size_t)(n0 + min(g + 8, nvalid - 1)) * K + k0 + t4 * 8;
  const int n = min(nch, npf);
  for (int c = 0; c < n; ++c) {
    cp_async16(pf + (2 * c) * 32 + lane, w0 + 32 * c);
    cp_async16(pf + (2 * c + 1) * 32 + lane, w1 + 32 * c);
  }
}

// Prefetch the round-0 weight fragments of a projection for this warp.
__device__ __forceinline__ void mg_prefetch_proj(const bf16* W, int N, int K, uint4* pf, int npf) {
  const MgSplit sp(N, K);
  const int tile = sp.tile(0);
  if (tile < sp.ntiles) mg_fetch(W, K, tile * 16, N - tile * 16, sp.kpart() * sp.cpw * 32, sp.cpw, pf, npf);
  cp_async_commit();
}
__device__ __forceinline__ void mg_prefetch_vocab(const MegaParams& p, uint4* pf) {
  const int tile = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  if (tile * 16 < p.V) mg_fetch(p.E, p.d, tile * 16, p.V - tile * 16, 0, p.d / 32, pf, p.npf);
  cp_async_commit();
}

// One warp: partial product of a 16-feature weight tile (rows n0.., [N][K]
// K-major) with NT n-tiles of activations over chunks [k0/32, k0/32 + nch):
// the first npf chunks come from the prefetch slot, the rest straight from
// L2/HBM in one batch. B operand: shared memory (act, ld ald) or, with GB, a
// bf16 global buffer written earlier in this launch (L2 loads).
// c[j][0..1] = feature n0+g, rows 8j+2t, 8j+2t+1; c[j][2..3] = feature n0+g+8.
template <int NT, bool GB>
__device__ __forceinline__ void mg_tile(const bf16* __restrict__ W, int K, int n0, int nvalid, int k0, int nch,
                                        const bf16* act, int ald, const uint4* pf, int npf, float (&c)[NT][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const bf16* a = act + (size_t)g * ald + k0 + t4 * 8;
  auto bfrag = [&](int j, int ch) -> uint4 {
    const bf16* q = a + (size_t)j * 8 * ald + 32 * ch;
    if (GB) return __ldcg(reinterpret_cast<const uint4*>(q));
    return *reinterpret_cast<const uint4*>(q);
  };
  float c2[NT][4];  // second accumulator chain (odd chunks)
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) c[j][e] = c2[j][e] = 0.f;
  const int np = min(nch, npf);
  auto from_slot = [&]() {
#pragma unroll
    for (int ch = 0; ch < 8; ch += 2) {
      if (ch < np) {
        const uint4 u0 = pf[(2 * ch) * 32 + lane], u1 = pf[(2 * ch + 1) * 32 + lane];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint4 v = bfrag(j, ch);
          mg_mma(c[j], u0.x, u1.x, u0.y, u1.y, v.x, v.y);
          mg_mma(c[j], u0.z, u1.z, u0.w, u1.w, v.z, v.w);
        }
      }
      if (ch + 1 < np) {
        const uint4 u0 = pf[(2 * ch + 2) * 32 + lane], u1 = pf[(2 * ch + 3) * 32 + lane];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint4 v = bfrag(j, ch + 1);
          mg_mma(c2[j], u0.x, u1.x, u0.y, u1.y, v.x, v.y);
          mg_mma(c2[j], u0.z, u1.z, u0.w, u1.w, v.z, v.w);
        }
      }
    }
  };
  const int nd = nch - np;
  if (nd <= 0) {
    from_slot();
  } else {
    // chunks the slot does not hold: one batch of direct loads issued before the slot math
    const bf16* w0 = W + (size_t)(n0 + min(g, nvalid - 1)) * K + k0 + t4 * 8;
    const bf16* w1 = W + (size_t)(n0 + min(g + 8, nvalid - 1)) * K + k0 + t4 * 8;
    constexpr int B = NT <= 2 ? 8 : 4;
    uint4 d0[B], d1[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int ch = np + (i < nd ? i : 0);  // unconditional (clamped) loads: no local-memory demotion
      d0[i] = ldw16(w0 + 32 * ch);
      d1[i] = ldw16(w1 + 32 * ch);
    }
    from_slot();
#pragma unroll
    for (int i = 0; i < B; ++i) {
      if (i < nd) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint4 v = bfrag(j, np + i);
          if (i & 1) {
            mg_mma(c2[j], d0[i].x, d1[i].x, d0[i].y, d1[i].y, v.x, v.y);
            mg_mma(c2[j], d0[i].z, d1[i].z, d0[i].w, d1[i].w, v.z, v.w);
          } else {
            mg_mma(c[j], d0[i].x, d1[i].x, d0[i].y, d1[i].y, v.x, v.y);
            mg_mma(c[j], d0[i].z, d1[i].z, d0[i].w, d1[i].w, v.z, v.w);
          }
        }
      }
    }
    for (int ch = np + B; ch < nch; ++ch) {  // only when the slot is shallow
      const uint4 u0 = ldw16(w0 + 32 * ch), u1 = ldw16(w1 + 32 * ch);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const uint4 v = bfrag(j, ch);
        mg_mma(c[j], u0.x, u1.x, u0.y, u1.y, v.x, v.y);
        mg_mma(c[j], u0.z, u1.z, u0.w, u1.w, v.z, v.w);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) c[j][e] += c2[j][e];
}

// Projection phase. epi(n, r, acc) for every valid (feature n < N, row r < R)
// of the tiles this warp finalises. red: shared scratch for split-K partials.
template <int NT, bool GB, class Epi>
__device__ __forceinline__ void mg_proj(const bf16* __restrict__ W, int N, int K, const bf16* act, int ald, int R,
                                        float* red, const uint4* pf, int npf, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const MgSplit sp(N, K);
  const int nr = sp.rounds(), kp = sp.kpart();
  for (int q = 0; q < nr; ++q) {
    const int tile = sp.tile(q);
    float c[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
    const bool valid = tile < sp.ntiles;
    if (valid)
      mg_tile<NT, GB>(W, K, tile * 16, N - tile * 16, kp * sp.cpw * 32, sp.cpw, act, ald, pf, q == 0 ? npf : 0, c);
    if (sp.kspl > 1) {  // deterministic split-K reduction through shared memory (fixed warp order)
      float* rp = red + (size_t)warp * (NT * 4 * 32);
      if (valid) {
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) rp[(j * 4 + e) * 32 + lane] = c[j][e];
      }
      __syncthreads();
      if (valid && kp == 0) {
        for (int w = warp + 1; w < warp + sp.kspl; ++w) {
          const float* o = red + (size_t)w * (NT * 4 * 32);
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) c[j][e] += o[(j * 4 + e) * 32 + lane];
        }
      }
      __syncthreads();
    }
    if (valid && kp == 0) {
      const int f0 = tile * 16 + g, f1 = f0 + 8;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int r0 = 8 * j + 2 * t4;
        if (r0 < R) {
          if (f0 < N) epi(f0, r0, c[j][0], q, j * 4 + 0);
          if (f1 < N) epi(f1, r0, c[j][2], q, j * 4 + 2);
        }
        if (r0 + 1 < R) {
          if (f0 < N) epi(f0, r0 + 1, c[j][1], q, j * 4 + 1);
          if (f1 < N) epi(f1, r0 + 1, c[j][3], q, j * 4 + 3);
        }
      }
    }
  }
}

// LayerNorm of one fp32 row held as float4 chunks (lane owns columns
// c*128 + lane*4 ..) -> bf16 row (population variance, eps 1e-5;
// kernels.py:42-57). Gain/bias are L1-resident constants.
__device__ __forceinline__ void mg_ln_row_store(const float4 (&v)[8], int nc, float inv_k, const float* g,
                                                const float* b, bf16* out) {
  const int lane = threadIdx.x & 31;
  float4 gq[8], bq[8];  // gain / bias loads issued before the reductions
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    gq[c] = c < nc ? __ldg(reinterpret_cast<const float4*>(g + c * 128 + lane * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    bq[c] = c < nc ? __ldg(reinterpret_cast<const float4*>(b + c * 128 + lane * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nc) s += (v[c].x + v[c].y) + (v[c].z + v[c].w);
  const float mean = warp_sum(s) * inv_k;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nc) {
      const float a = v[c].x - mean, bb = v[c].y - mean, cc = v[c].z - mean, dd = v[c].w - mean;
      q += a * a + bb * bb + cc * cc + dd * dd;
    }
  const float inv = rsqrtf(warp_sum(q) * inv_k + 1e-5f);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nc) {
      const int j = c * 128 + lane * 4;
      const float4 gv = gq[c], bv = bq[c];
      __nv_bfloat162 lo = __floats2bfloat162_rn((v[c].x - mean) * inv * gv.x + bv.x, (v[c].y - mean) * inv * gv.y + bv.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn((v[c].z - mean) * inv * gv.z + bv.z, (v[c].w - mean) * inv * gv.w + bv.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(out + j) = u;
    }
}

// Stage LN(x) for R rows into bf16 shared memory (one warp per row).
__device__ __forceinline__ void mg_stage_ln(const float* src, int R, int K, const float* g, const float* b, bf16* act,
                                            int ald) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nc = K / 128;
  for (int r = warp; r < R; r += MG_WARPS) {
    const float* xr = src + (size_t)r * K;
    float4 v[8];  // K <= 1024
#pragma unroll
    for (int c = 0; c < 8; ++c)
      v[c] = c < nc ? __ldcg(reinterpret_cast<const float4*>(xr + c * 128 + lane * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    mg_ln_row_store(v, nc, __fdividef(1.0f, (float)K), g, b, act + (size_t)r * ald);
  }
  __syncthreads();
}

// online {max, sum exp} + top-1 (value desc, id asc) over the generable set
struct MgStat {
  float mx, sum, bv;
  int bi;
  __device__ __forceinline__ void init() {
    mx = -INFINITY;
    sum = 0.f;
    bv = -INFINITY;
    bi = 0x7fffffff;
  }
  __device__ __forceinline__ void add(float l, int v) {
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
  __device__ __forceinline__ void merge(float om, float os, float obv, int obi) {
    if (om != -INFINITY) {
      const float m = fmaxf(mx, om);
      sum = (mx == -INFINITY ? 0.f : sum * ex2f((mx - m) * LOG2E)) + os * ex2f((om - m) * LOG2E);
      mx = m;
    }
    if (better(obv, obi, bv, bi)) {
      bv = obv;
      bi = obi;
    }
  }
};

// ---------------------------------------------------------------------------
// Selection of step t for row r (decoding.py:102-150, beam = 1) by one warp:
// merges the grid's vocab partials in a fixed order (every caller gets the
// same token); the writer also updates the row's decoding state.
// Returns the token fed at step t + 1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int mg_select_row(const MegaParams& p, int r, int t, bool writer) {
  const int lane = threadIdx.x & 31;
  const GreedyState& st = p.st;
  const int feed = __ldcg(st.feed + r), done = __ldcg(st.done + r), cap = st.caps[r];
  const float eos = __ldcg(p.veos + r);
  MgStat s;
  s.init();
  for (int b = lane; b < gridDim.x; b += 32) {
    const float4 v = __ldcg(p.vpart + (size_t)r * gridDim.x + b);
    s.merge(v.x, v.y, v.z, __float_as_int(v.w));
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, s.mx, o);
    const float os = __shfl_xor_sync(0xffffffffu, s.sum, o);
    const float ov = __shfl_xor_sync(0xffffffffu, s.bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, s.bi, o);
    s.merge(om, os, ov, oi);
  }
  if (done) return feed;  // finished rows keep feeding EOS (outputs ignored)
  const bool last = (t == cap - 1);
  float bv = s.bv;
  int bi = s.bi;
  if (bi == 0x7fffffff) {  // non-finite logits: finish the row rather than emit a bogus id
    bi = EOS_ID;
    bv = eos;
  }
  const int tok = last ? EOS_ID : bi;
  if (writer && lane == 0) {
    const float logit = last ? eos : bv;
    const float lp = (logit - s.mx) - logf(s.sum);
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
  return tok;
}

// ---------------------------------------------------------------------------
// phases
// ---------------------------------------------------------------------------
// A: [selection of step t-1 + embedding] [LN1] QKV of layer i; K/V appended at slot t.
// sel_prev: rows [0, R_prev) have vocab partials of step t-1 to select from.
template <int NT>
__device__ __noinline__ void mg_ph_qkv(const MegaParams& p, int i, int t, int R, int R_prev, bool sel_prev,
                                          bf16* act, float* red, uint4* pf) {
  const int d = p.d, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const MegaLayer& W = p.L[i];
  const size_t lay = (size_t)i * p.rcap * p.cap * d;
  const MgSplit sp(3 * d, d);
  const bool work = sp.cta_has_work();
  const int nc = d / 128;
  if (sel_prev) {
    // rows this CTA stages (all live rows, if it has QKV work) or owns the state of (r % grid == blockIdx)
    if (warp < R_prev) {
      for (int r = warp; r < R_prev; r += MG_WARPS) {
        const bool stage = work && r < R;
        const bool writer = (r % gridDim.x) == (int)blockIdx.x;
        if (!stage && !writer) continue;
        float4 pp[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)  // positional row of the next input, issued before the merge
          pp[c] = c < nc ? __ldg(reinterpret_cast<const float4*>(p.pe + (size_t)t * p.k * d + c * 128 + lane * 4))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        const int tok = mg_select_row(p, r, t - 1, writer);
        if (r < R) {
          // x = E[tok] * sqrt(d) + PE[t k] (fp32, unfused mul/add as the reference)
          float4 v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c < nc) {
              const uint2 u = __ldg(reinterpret_cast<const uint2*>(p.E + (size_t)tok * d + c * 128 + lane * 4));
              const float2 e0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
              const float2 e1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
              v[c] = make_float4(__fadd_rn(__fmul_rn(e0.x, p.scale), pp[c].x),
                                 __fadd_rn(__fmul_rn(e0.y, p.scale), pp[c].y),
                                 __fadd_rn(__fmul_rn(e1.x, p.scale), pp[c].z),
                                 __fadd_rn(__fmul_rn(e1.y, p.scale), pp[c].w));
            } else {
              v[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          if (writer)
            for (int c = 0; c < nc; ++c) *reinterpret_cast<float4*>(p.x + (size_t)r * d + c * 128 + lane * 4) = v[c];
          if (stage) mg_ln_row_store(v, nc, __fdividef(1.0f, (float)d), W.ln1g, W.ln1b, act + (size_t)r * (d + MG_APAD));
        }
      }
    }
    __syncthreads();
  } else if (work) {
    mg_stage_ln(p.x, R, d, W.ln1g, W.ln1b, act, d + MG_APAD);
  }
  if (!work) return;
  cp_async_wait_all();
  mg_proj<NT, false>(W.wqkv, 3 * d, d, act, d + MG_APAD, R, red, pf, p.npf, [&](int n, int r, float acc, int, int) {
    const bf16 v = __float2bfloat16_rn(acc + __ldg(W.bqkv + n));
    if (n < d)
      p.q[(size_t)r * d + n] = v;
    else if (n < 2 * d)
      p.kc[lay + ((size_t)r * p.cap + t) * d + (n - d)] = v;
    else
      p.vc[lay + ((size_t)r * p.cap + t) * d + (n - 2 * d)] = v;
  });
}

// D / G: LN(x) -> bf16 out (N = d or ff, optional ReLU): Qc (infer.py:272) / W1 (infer.py:287-289)
template <int NT, bool RELU>
__device__ __noinline__ void mg_ph_ln_proj(const MegaParams& p, const float* g, const float* b, const bf16* W,
                                              const float* bias, int N, bf16* out, int R, bf16* act, float* red,
                                              uint4* pf) {
  const int d = p.d;
  if (!MgSplit(N, d).cta_has_work()) return;
  mg_stage_ln(p.x, R, d, g, b, act, d + MG_APAD);
  cp_async_wait_all();
  mg_proj<NT, false>(W, N, d, act, d + MG_APAD, R, red, pf, p.npf, [&](int n, int r, float acc, int, int) {
    float v = acc + __ldg(bias + n);
    if (RELU) v = fmaxf(v, 0.f);
    out[(size_t)r * N + n] = __float2bfloat16_rn(v);
  });
}

// Stage R rows of a bf16 global buffer (ld K, written by other CTAs this launch) into act.
__device__ __forceinline__ void mg_stage_copy(const bf16* src, int R, int K, bf16* act, int ald) {
  const int per = K / 8, n = R * per;
  constexpr int U = 4;  // loads in flight per thread before the stores
  for (int i0 = threadIdx.x; i0 < n; i0 += MG_THREADS * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = min(i0 + u * MG_THREADS, n - 1);
      const int r = i / per, c = (i - r * per) * 8;
      v[u] = __ldcg(reinterpret_cast<const uint4*>(src + (size_t)r * K + c));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * MG_THREADS;
      if (i < n) {
        const int r = i / per, c = (i - r * per) * 8;
        *reinterpret_cast<uint4*>(act + (size_t)r * ald + c) = v[u];
      }
    }
  }
  __syncthreads();
}

// C / F / H: x += src @ W^T + bias  (Wo / Woc / W2 + residual, infer.py:204-205, :284-285, :290-292)
template <int NT>
__device__ __noinline__ void mg_ph_residual(const MegaParams& p, const bf16* src, int K, const bf16* W,
                                            const float* bias, int R, bf16* act, float* red, uint4* pf) {
  const int d = p.d;
  const MgSplit sp(d, K);
  if (!sp.cta_has_work()) return;
  // residual and bias operands of this lane's round-0 outputs, loaded before the staging round trip
  float xr[NT * 4], br[2];
  {
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int tile = sp.tile(0);
    const bool own = tile < sp.ntiles && sp.kpart() == 0;
    const int f0 = min(tile * 16 + g, d - 1), f1 = min(tile * 16 + g + 8, d - 1);
    br[0] = own ? __ldg(bias + f0) : 0.f;
    br[1] = own ? __ldg(bias + f1) : 0.f;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int r0 = min(8 * j + 2 * t4, R - 1), r1 = min(8 * j + 2 * t4 + 1, R - 1);
      xr[j * 4 + 0] = own ? __ldcg(p.x + (size_t)r0 * d + f0) : 0.f;
      xr[j * 4 + 1] = own ? __ldcg(p.x + (size_t)r1 * d + f0) : 0.f;
      xr[j * 4 + 2] = own ? __ldcg(p.x + (size_t)r0 * d + f1) : 0.f;
      xr[j * 4 + 3] = own ? __ldcg(p.x + (size_t)r1 * d + f1) : 0.f;
    }
  }
  mg_stage_copy(src, R, K, act, K + MG_APAD);
  cp_async_wait_all();
  mg_proj<NT, false>(W, d, K, act, K + MG_APAD, R, red, pf, p.npf, [&](int n, int r, float acc, int q, int slot) {
    float* xp = p.x + (size_t)r * d + n;
    if (q == 0)
      *xp = xr[slot] + (acc + br[slot >> 1 & 1]);
    else
      *xp = __ldcg(xp) + (acc + __ldg(bias + n));
  });
}

// B / E: decode attention (infer.py:259-285), dh = 64. Item (row, head) ->
// CTA (item % grid), warp group (item / grid) of MG_AWARPS warps; warp w of
// the group takes keys w*32 + lane (+ 256 m): scores with one key per lane,
// PV with two head dims per lane (the lane's weights broadcast by shuffle),
// online softmax across rounds; the group merges {max, sum, out} through
// shared memory.
template <bool SELF>
__device__ __noinline__ void mg_ph_attn(const MegaParams& p, int layer, int t, int R, float* scratch) {
  constexpr int DH = 64;
  const int d = p.d, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ngrp = MG_WARPS / MG_AWARPS, grp = warp / MG_AWARPS, wk = warp % MG_AWARPS;
  const int items = R * p.H;
  const int nr = (items + gridDim.x * ngrp - 1) / (gridDim.x * ngrp);
  float* qsm = scratch + (size_t)warp * (DH + 66);  // per warp: q[64], then {out[64], m, l}
  float* sp = qsm + DH;
  for (int q = 0; q < nr; ++q) {
    const int it = blockIdx.x + gridDim.x * (grp + ngrp * q);
    const bool valid = it < items;
    if (valid) {
      const int r = it / p.H, h = it - r * p.H;
      const bf16* kbase;
      const bf16* vbase;
      size_t rs;
      int L;
      if (SELF) {
        const size_t lay = (size_t)layer * p.rcap * p.cap * d + (size_t)r * p.cap * d + h * DH;
        kbase = p.kc + lay;
        vbase = p.vc + lay;
        rs = d;
        L = t + 1;
      } else {
        const size_t o = (size_t)p.src_off[r] * p.xstride + (size_t)2 * layer * d + h * DH;
        kbase = p.xkv + o;
        vbase = p.xkv + o + d;
        rs = p.xstride;
        L = p.src_len[r];
      }
      {
        const __nv_bfloat162 q2 = __ldcg(reinterpret_cast<const __nv_bfloat162*>(p.q + (size_t)r * d + h * DH + 2 * lane));
        const float2 f = __bfloat1622float2(q2);
        qsm[2 * lane] = f.x * p.att_scale;
        qsm[2 * lane + 1] = f.y * p.att_scale;
      }
      __syncwarp();
      float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f;
      for (int j0 = wk * 32; j0 < L; j0 += MG_AWARPS * 32) {
        const int j = j0 + lane;
        const int jj = j < L ? j : L - 1;
        uint4 kr[8];
        uint32_t vr[32];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          kr[c] = SELF ? __ldcg(reinterpret_cast<const uint4*>(kbase + (size_t)jj * rs + c * 8))
                       : __ldg(reinterpret_cast<const uint4*>(kbase + (size_t)jj * rs + c * 8));
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int jv = min(j0 + i, L - 1);
          const uint32_t* vp = reinterpret_cast<const uint32_t*>(vbase + (size_t)jv * rs + 2 * lane);
          vr[i] = SELF ? __ldcg(vp) : __ldg(vp);
        }
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const __nv_bfloat162* hk = reinterpret_cast<const __nv_bfloat162*>(&kr[c]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(hk[e]);
            a0 = fmaf(qsm[c * 8 + 2 * e], f.x, a0);
            a1 = fmaf(qsm[c * 8 + 2 * e + 1], f.y, a1);
          }
        }
        const float s = j < L ? a0 + a1 : -INFINITY;
        const float mn = fmaxf(m, warp_max(s));
        const float sc = ex2f((m - mn) * LOG2E);  // first round: m = -inf -> sc = 0
        const float pj = j < L ? ex2f((s - mn) * LOG2E) : 0.f;
        l = l * sc + warp_sum(pj);
        m = mn;
        o0 *= sc;
        o1 *= sc;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float pi = __shfl_sync(0xffffffffu, pj, i);  // 0 for keys >= L
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vr[i]));
          o0 = fmaf(pi, f.x, o0);
          o1 = fmaf(pi, f.y, o1);
        }
      }
      sp[2 * lane] = o0;
      sp[2 * lane + 1] = o1;
      if (lane == 0) {
        sp[64] = m;
        sp[65] = l;
      }
    }
    __syncthreads();
    if (valid && wk == 0) {
      const int r = it / p.H, h = it - r * p.H;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < MG_AWARPS; ++w) M = fmaxf(M, scratch[(size_t)(grp * MG_AWARPS + w) * (DH + 66) + DH + 64]);
      float Lsum = 0.f, a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int w = 0; w < MG_AWARPS; ++w) {
        const float* g0 = scratch + (size_t)(grp * MG_AWARPS + w) * (DH + 66) + DH;
        const float mw = g0[64];
        if (mw != -INFINITY) {
          const float f = ex2f((mw - M) * LOG2E);
          Lsum += g0[65] * f;
          a0 += g0[2 * lane] * f;
          a1 += g0[2 * lane + 1] * f;
        }
      }
      const float inv = 1.0f / Lsum;
      *reinterpret_cast<__nv_bfloat162*>(p.ctx + (size_t)r * d + h * DH + 2 * lane) =
          __floats2bfloat162_rn(a0 * inv, a1 * inv);
    }
    __syncthreads();
  }
}

// I: vocabulary statistics (Stage-I normaliser over the full vocabulary,
// infer.py:293-301; top-1 over the generable set, decoding.py:84-87, :112):
// warps own whole 16-column tiles of E (spread across SMs first); per-CTA
// partials land in vpart[row][blockIdx].
template <int NT>
__device__ __noinline__ void mg_ph_vocab(const MegaParams& p, int R, bf16* act, float* red, uint4* pf) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  mg_stage_ln(p.x, R, p.d, p.lng, p.lnb, act, p.d + MG_APAD);
  cp_async_wait_all();
  const int ald = p.d + MG_APAD;
  const int ntiles = (p.V + 15) / 16;
  const int GW = gridDim.x * MG_WARPS;
  MgStat st[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) st[j][0].init(), st[j][1].init();
  bool first = true;
  for (int tile = warp * gridDim.x + blockIdx.x; tile < ntiles; tile += GW) {
    float c[NT][4];
    const int n0 = tile * 16;
    mg_tile<NT, false>(p.E, p.d, n0, p.V - n0, 0, p.d / 32, act, ald, pf, first ? p.npf : 0, c);
    first = false;
    const int f0 = n0 + g, f1 = n0 + g + 8;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (f0 < p.V) {
        st[j][0].add(c[j][0], f0);
        st[j][1].add(c[j][1], f0);
      }
      if (f1 < p.V) {
        st[j][0].add(c[j][2], f1);
        st[j][1].add(c[j][3], f1);
      }
      if (f0 == EOS_ID) {
        if (8 * j + 2 * t4 < R) p.veos[8 * j + 2 * t4] = c[j][0];
        if (8 * j + 2 * t4 + 1 < R) p.veos[8 * j + 2 * t4 + 1] = c[j][1];
      }
    }
  }
  // merge the 8 lanes (g) that share rows, then the 16 warps through shared memory
  float4* ws = reinterpret_cast<float4*>(red);  // [warps][MG_RMAX]
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      MgStat& s = st[j][e];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, s.mx, o);
        const float os = __shfl_xor_sync(0xffffffffu, s.sum, o);
        const float ov = __shfl_xor_sync(0xffffffffu, s.bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, s.bi, o);
        s.merge(om, os, ov, oi);
      }
      if (g == 0) ws[warp * MG_RMAX + 8 * j + 2 * t4 + e] = make_float4(s.mx, s.sum, s.bv, __int_as_float(s.bi));
    }
  __syncthreads();
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    MgStat s;
    s.init();
    for (int w = 0; w < MG_WARPS; ++w) {
      const float4 v = ws[w * MG_RMAX + r];
      s.merge(v.x, v.y, v.z, __float_as_int(v.w));
    }
    p.vpart[(size_t)r * gridDim.x + blockIdx.x] = make_float4(s.mx, s.sum, s.bv, __int_as_float(s.bi));
  }
}

// final selection after the last computed step (state only)
__device__ __noinline__ void mg_ph_select_last(const MegaParams& p, int t, int R) {
  const int warp = threadIdx.x >> 5;
  for (int r = warp; r < R; r += MG_WARPS)
    if ((r % gridDim.x) == (int)blockIdx.x) mg_select_row(p, r, t, true);
}

struct MgCtx {
  unsigned target;
  int tr_i;
};

// grid barrier with the next phase's weight prefetch issued between arrive and wait
template <class Pf>
__device__ __forceinline__ void mg_barrier(const MegaParams& p, int t, MgCtx& c, Pf prefetch) {
  mg_arrive(p.bar);
  prefetch();
  c.target += gridDim.x;
  mg_wait(p.bar, c.target);
  if (p.trace && t == p.trace_step && blockIdx.x == 0 && threadIdx.x == 0 && c.tr_i < 63)
    p.trace[c.tr_i++] = mg_clock();
}

template <int NT>
__device__ __noinline__ void mg_step(const MegaParams& p, int t, int R, int R_prev, bf16* act, float* red, uint4* pf,
                                     MgCtx& c) {
  const int d = p.d, ff = p.ff, npf = p.npf;
  if (p.trace && t == p.trace_step && blockIdx.x == 0 && threadIdx.x == 0 && c.tr_i < 63) p.trace[c.tr_i++] = mg_clock();
  auto none = [] {};
  for (int i = 0; i < p.Ld; ++i) {
    const MegaLayer& W = p.L[i];
    const int sk = p.skip;
    if (!(sk & 1)) mg_ph_qkv<NT>(p, i, t, R, R_prev, i == 0 && t > p.t_begin, act, red, pf);  // A
    mg_barrier(p, t, c, [&] { mg_prefetch_proj(W.wo, d, d, pf, npf); });
    if (!(sk & 2)) mg_ph_attn<true>(p, i, t, R, red);  // B: self attention over slots 0..t
    mg_barrier(p, t, c, none);
    if (!(sk & 4)) mg_ph_residual<NT>(p, p.ctx, d, W.wo, W.bo, R, act, red, pf);  // C: Wo + residual
    mg_barrier(p, t, c, [&] { mg_prefetch_proj(W.wqc, d, d, pf, npf); });
    if (!(sk & 8)) mg_ph_ln_proj<NT, false>(p, W.ln2g, W.ln2b, W.wqc, W.bqc, d, p.q, R, act, red, pf);  // D: [LN2] Qc
    mg_barrier(p, t, c, [&] { mg_prefetch_proj(W.woc, d, d, pf, npf); });
    if (!(sk & 16)) mg_ph_attn<false>(p, i, t, R, red);  // E: cross attention over the source
    mg_barrier(p, t, c, none);
    if (!(sk & 32)) mg_ph_residual<NT>(p, p.ctx, d, W.woc, W.boc, R, act, red, pf);  // F: Woc + residual
    mg_barrier(p, t, c, [&] { mg_prefetch_proj(W.w1, ff, d, pf, npf); });
    if (!(sk & 64)) mg_ph_ln_proj<NT, true>(p, W.ln3g, W.ln3b, W.w1, W.b1, ff, p.hid, R, act, red, pf);  // G: [LN3] W1
    mg_barrier(p, t, c, [&] { mg_prefetch_proj(W.w2, d, ff, pf, npf); });
    if (!(sk & 128)) mg_ph_residual<NT>(p, p.hid, ff, W.w2, W.b2, R, act, red, pf);  // H: W2 + residual
    if (i + 1 < p.Ld)
      mg_barrier(p, t, c, [&] { mg_prefetch_proj(p.L[i + 1].wqkv, 3 * d, d, pf, npf); });
    else
      mg_barrier(p, t, c, [&] { mg_prefetch_vocab(p, pf); });
  }
  if (!(p.skip & 256)) mg_ph_vocab<NT>(p, R, act, red, pf);  // I: [final LN] vocabulary statistics
  mg_barrier(p, t, c, [&] { mg_prefetch_proj(p.L[0].wqkv, 3 * d, d, pf, npf); });
}

__global__ void __launch_bounds__(MG_THREADS, 1) decode_mega_kernel(const __grid_constant__ MegaParams p) {
  extern __shared__ __align__(16) unsigned char msm_raw[];
  uint4* pf = reinterpret_cast<uint4*>(msm_raw) + (size_t)(threadIdx.x >> 5) * p.npf * 64;  // per-warp weight slot
  bf16* act = reinterpret_cast<bf16*>(reinterpret_cast<uint4*>(msm_raw) + (size_t)MG_WARPS * p.npf * 64);
  float* red = reinterpret_cast<float*>(act + (size_t)MG_RMAX * ((p.ff > p.d ? p.ff : p.d) + MG_APAD));
  MgCtx c{0u, 0};
  mg_prefetch_proj(p.L[0].wqkv, 3 * p.d, p.d, pf, p.npf);
  int R_prev = 0, t_last = -1;
  for (int t = p.t_begin; t < p.t_end; ++t) {
    const int R = p.alive[t];
    if (R <= 0) break;
    // finished is updated in phase A (one step behind): this sees rows done by step t-2
    if (__ldcg(&p.ctl->finished) >= p.nrows) break;
    if (R <= 8)
      mg_step<1>(p, t, R, R_prev, act, red, pf, c);
    else
      mg_step<2>(p, t, R, R_prev, act, red, pf, c);
    R_prev = R;
    t_last = t;
  }
  cp_async_wait_all();
  if (t_last >= 0) mg_ph_select_last(p, t_last, R_prev);
}

// shared memory: prefetch slots + activations [MG_RMAX][max(d, ff) + pad] + scratch
// (split-K partials / vocab warp stats / attention group merge)
inline size_t mega_red_floats() {
  const size_t a = (size_t)MG_WARPS * 2 * 4 * 32;   // split-K partials (NT <= 2)
  const size_t b = (size_t)MG_WARPS * MG_RMAX * 4;  // vocab warp stats
  const size_t c = (size_t)MG_WARPS * (64 + 66);    // attention q + merge
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}
inline size_t mega_smem_bytes(int d, int ff, int npf) {
  const int kmax = ff > d ? ff : d;
  return (size_t)MG_WARPS * npf * 64 * 16 + (size_t)MG_RMAX * (kmax + MG_APAD) * sizeof(bf16) +
         mega_red_floats() * sizeof(float);
}

}  // namespace hrt
