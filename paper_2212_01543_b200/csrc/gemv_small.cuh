// Small-M projections ("GEMV" regime) on mma.sync for the latency-bound
// shapes: Stage-I decode steps at small live-row counts and the encoder /
// Stage II at batch 1 (M <= 32 rows).
//
//     C[M, N] = A[M, K] . W[N, K]^T   (bf16 in, fp32 accumulate)
//
// At these shapes the tcgen05 tile (128 x BN, one TMA pipeline per CTA over
// the whole K) leaves a handful of CTAs each streaming its weight panel
// serially; here one CTA owns 16 output features and its 16 warps split K, so
// every weight byte is requested by its own lane at kernel start (before the
// PDL grid-dependency wait: weights never depend on the previous kernel).
// Swap-AB mma.sync m16n8k16: the 16-feature weight tile is the M side, the
// rows (8 per n-tile) the N side; the K index is permuted identically on both
// operands (lane (g, t) holds k = 8t..8t+7 of each 32-wide chunk) so each
// weight fragment is one 16-byte load. Partial sums are reduced across warps
// in shared memory in a fixed order (deterministic), then warp 0 runs the
// same element-wise epilogue functors as the tcgen05 GEMM (gemm_epi.cuh).
//
// gemv_vocab_kernel: the tied vocabulary projection (infer.py:293-301) with
// the Stage-I statistics fused: a CTA covers 256 columns (16 warps x 16) and
// emits one {max, sum exp, top-1 allowed} partial per row, in the VocabParts
// layout the selection kernels merge.
#pragma once
#include "common.cuh"
#include "gemm_epi.cuh"
#include "kernels.cuh"

namespace hrt {

constexpr int GV_WARPS = 16;
constexpr int GV_THREADS = GV_WARPS * 32;
constexpr int GV_MAXC = 8;  // K-chunks (32 wide) per warp held in registers (K <= 4096)

__device__ __forceinline__ void gv_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// weight fragment load: read-only path, no L1 allocation, L2 evict-last (the
// decoder + vocabulary weights, ~40 MB in bf16, stay L2-resident across steps)
__device__ __forceinline__ uint64_t gv_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 gv_ldw(const bf16* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Fragment-native weight copy for the GEMV kernels. For output-feature group
// q (16 rows), 32-wide K chunk ch and half u (rows g / g + 8), the 32 lanes'
// 16-byte fragments (lane (g, t): row 16 q + g + 8 u, k = 32 ch + 8 t .. + 8)
// are stored as one contiguous 512-byte run, so every weight load instruction
// of a warp reads 512 contiguous bytes instead of 8 rows x 64 bytes (the
// row-major pattern measured 2x slower to stream out of L2). Rows past N are
// zero. Size: cdiv(N, 16) * 16 * K elements.
__host__ __device__ constexpr size_t gv_frag_elems(int N, int K) { return (size_t)((N + 15) / 16) * 16 * K; }
__global__ void gv_frag_layout_kernel(const bf16* __restrict__ W, int N, int K, bf16* __restrict__ out) {
  const int nch = K / 32;
  const size_t total = (size_t)((N + 15) / 16) * nch * 2 * 32;  // 16-byte fragments
  for (size_t f = (size_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += (size_t)gridDim.x * blockDim.x) {
    const int lane = (int)(f & 31);
    const size_t blk = f >> 5;  // (grp * nch + ch) * 2 + u
    const int u = (int)(blk & 1);
    const size_t gc = blk >> 1;
    const int ch = (int)(gc % nch);
    const size_t grp = gc / nch;
    const size_t row = grp * 16 + (lane >> 2) + 8 * u;
    const int col = 32 * ch + 8 * (lane & 3);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < (size_t)N) v = *reinterpret_cast<const uint4*>(W + row * K + col);
    *reinterpret_cast<uint4*>(out + f * 8) = v;
  }
}
// base of feature group n0 / 16 in a fragment-native copy; fragment (ch, u) of lane at + ((2 ch + u) * 32 + lane) * 8
__device__ __forceinline__ const bf16* gv_frag_group(const bf16* Wf, int n0, int K) {
  return Wf + (size_t)(n0 >> 4) * (K / 32) * 2 * 256;
}

// Optional LayerNorm prologue (the activation operand is LN(x) of fp32 rows,
// kernels.py:42-57): the CTA computes every row's statistics exactly as
// layernorm_vec_kernel does (same lane partition and reduction order, so the
// bf16 operand is bit-identical to the unfused LN kernel's output) and
// normalises the 8-element fragments it feeds the MMA.
struct GvLN {
  const float* x;  // [M][K] fp32 rows (nullptr: A is the bf16 operand)
  const float* g;
  const float* b;
};

__device__ __forceinline__ void gv_ln_stats(const GvLN& ln, int M, int K, float2* st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = K / 128;
  for (int r = warp; r < M; r += (int)(blockDim.x >> 5)) {
    const float4* xr = reinterpret_cast<const float4*>(ln.x + (size_t)r * K);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < nv ? xr[lane + 32 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = warp_sum(s) / K;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) {
        const float a = v[i].x - mean, bb = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
        q += (a * a + bb * bb) + (c * c + e * e);
      }
    const float inv = 1.0f / sqrtf(warp_sum(q) / K + 1e-5f);
    if (lane == 0) st[r] = make_float2(mean, inv);
  }
}

// bf16 operand fragment: 8 consecutive k of row r (LN applied when ln.x != nullptr)
template <bool LNA>
__device__ __forceinline__ uint4 gv_afrag(const bf16* A, int lda, const GvLN& ln, const float2* st, int K, int r,
                                          int k0) {
  if (!LNA) return *reinterpret_cast<const uint4*>(A + (size_t)r * lda + k0);
  const float4* xp = reinterpret_cast<const float4*>(ln.x + (size_t)r * K + k0);
  const float4* gp = reinterpret_cast<const float4*>(ln.g + k0);
  const float4* bp = reinterpret_cast<const float4*>(ln.b + k0);
  const float2 mi = st[r];
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float4 x = xp[h], g = __ldg(gp + h), b = __ldg(bp + h);
    __nv_bfloat162 lo = __floats2bfloat162_rn((x.x - mi.x) * mi.y * g.x + b.x, (x.y - mi.x) * mi.y * g.y + b.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn((x.z - mi.x) * mi.y * g.z + b.z, (x.w - mi.x) * mi.y * g.w + b.w);
    w[2 * h] = *reinterpret_cast<uint32_t*>(&lo);
    w[2 * h + 1] = *reinterpret_cast<uint32_t*>(&hi);
  }
  return u;
}

// Optional LayerNorm tail (residual projections): the last CTA to finish
// (arrival counter) normalises the M updated rows of x into y, exactly as
// layernorm_vec_kernel does, so the separate LN launch disappears.
struct GvTailLN {
  const float* g;  // nullptr: no tail
  const float* b;
  bf16* y;
  int* counter;  // zero between launches (the last CTA re-arms it)
};

__device__ __forceinline__ void gv_tail_ln(const float* x, int M, int K, const GvTailLN& t) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(t.counter, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = K / 128;
  for (int r = warp; r < M; r += GV_WARPS) {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)r * K);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < nv ? __ldcg(xr + lane + 32 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = warp_sum(s) / K;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) {
        const float a = v[i].x - mean, bb = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
        q += (a * a + bb * bb) + (c * c + e * e);
      }
    const float inv = 1.0f / sqrtf(warp_sum(q) / K + 1e-5f);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) {
        const int c4 = (lane + 32 * i) * 4;
        const float4 gg = *reinterpret_cast<const float4*>(t.g + c4);
        const float4 bv = *reinterpret_cast<const float4*>(t.b + c4);
        float4 o;
        o.x = (v[i].x - mean) * inv * gg.x + bv.x;
        o.y = (v[i].y - mean) * inv * gg.y + bv.y;
        o.z = (v[i].z - mean) * inv * gg.z + bv.z;
        o.w = (v[i].w - mean) * inv * gg.w + bv.w;
        __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(t.y + (size_t)r * K + c4) = u;
      }
  }
  if (threadIdx.x == 0) *t.counter = 0;  // re-arm for the next launch / graph replay
}

// Row blocks: blockIdx.y takes rows 8 NT y .. 8 NT (y + 1) - 1 (one weight pass per row
// block; the weights are L2-resident), so one launch covers up to gridDim.y x 8 NT rows.
template <int NT, int CPW, class Epi, bool LNA = false, bool TLN = false>
__global__ void __launch_bounds__(GV_THREADS) gemv_small_kernel(const bf16* __restrict__ A, int lda,
                                                                const bf16* __restrict__ W, int N, int K, int M,
                                                                const int* __restrict__ M_dev, Epi epi, GvLN ln,
                                                                GvTailLN tln) {
  constexpr int NG = NT < 4 ? NT : 4;  // n-tiles reduced per shared-memory pass
  __shared__ float red[GV_WARPS][NG * 4][32];
  __shared__ float2 lnst[LNA ? 8 * NT : 1];
  pdl_trigger();
  const int rb0 = blockIdx.y * 8 * NT;  // first row of this row block (0 without row blocking)
  A += (size_t)rb0 * lda;
  M -= rb0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int n0 = blockIdx.x * 16;
  const int nch = K / 32;  // == GV_WARPS * CPW, or fewer chunks than warps with CPW == 1
  const int c0 = warp * CPW, c1 = min(c0 + CPW, nch);
  const int nvalid = N - n0;
  (void)nvalid;
  // W is the fragment-native copy (gv_frag_layout_kernel): rows past N are zero
  const bf16* wf = gv_frag_group(W, n0, K) + lane * 8;
  // weight fragments: unconditional (clamped) loads keep the arrays in registers
  const uint64_t pol = gv_policy();
  uint4 u0[CPW], u1[CPW];
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    const int ch = min(c0 + i, nch - 1);
    u0[i] = gv_ldw(wf + (size_t)(2 * ch) * 256, pol);
    u1[i] = gv_ldw(wf + (size_t)(2 * ch + 1) * 256, pol);
  }
  pdl_wait();
  // Activation fragments do not depend on the live row count: for the small
  // shapes they are requested before the device row count resolves (rows
  // clamped to the launch's host bound, which the buffer always holds; rows
  // past the live count are computed and discarded) -- one dependent round
  // trip fewer on the critical path.
  constexpr bool HOIST = !LNA && CPW * NT <= 8;
  uint4 av[HOIST ? CPW : 1][HOIST ? NT : 1];
  if constexpr (HOIST) {
    const int m_host = M;
#pragma unroll
    for (int i = 0; i < CPW; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j)
        av[i][j] = c0 + i < c1 ? *reinterpret_cast<const uint4*>(A + (size_t)min(8 * j + g, m_host - 1) * lda +
                                                                  32 * (c0 + i) + t4 * 8)
                               : make_uint4(0, 0, 0, 0);
  }
  if (M_dev) M = *M_dev - rb0;
  if (M <= 0) return;  // every Stage-I row finished / no live row in this block (uniform across the CTA)
  // The final reduction and epilogue are spread over NG warps: warp w < NG owns
  // n-tiles w, w + NG, ...; its epilogue operands (residual rows, bias) are
  // issued now and consumed after the reduction.
  constexpr int NOWN = NT / NG;
  const bool owner = warp < NG;
  const int f0 = n0 + g, f1 = f0 + 8;
  float2 pre[NOWN][4];
  if (owner) {
#pragma unroll
    for (int o = 0; o < NOWN; ++o) {
      const int j = o * NG + warp;
      const int r0 = 8 * j + 2 * t4;
      const int ra = min(r0, M - 1), rb = min(r0 + 1, M - 1);
      const int fa = min(f0, N - 1), fb = min(f1, N - 1);
      pre[o][0] = epi.load2(rb0 + ra, fa);
      pre[o][1] = epi.load2(rb0 + rb, fa);
      pre[o][2] = epi.load2(rb0 + ra, fb);
      pre[o][3] = epi.load2(rb0 + rb, fb);
    }
  }
  if (LNA) {
    gv_ln_stats(ln, M, K, lnst);
    __syncthreads();
  }
  float c[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  // activation (B) fragments: row 8j+g, k = 32 ch + 8 t (n-tiles past M skipped)
  const int nt_live = min(NT, (M + 7) / 8);
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    if (c0 + i < c1) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        if (j < nt_live) {
          uint4 v;
          if constexpr (HOIST) {
            v = av[i][j];
          } else {
            const int r = min(8 * j + g, M - 1);
            v = gv_afrag<LNA>(A, lda, ln, lnst, K, r, 32 * (c0 + i) + t4 * 8);
          }
          gv_mma(c[j], u0[i].x, u1[i].x, u0[i].y, u1[i].y, v.x, v.y);
          gv_mma(c[j], u0[i].z, u1[i].z, u0[i].w, u1[i].w, v.z, v.w);
        }
      }
    }
  }
  // fixed-order reduction over the warps, NG n-tiles per pass
  float fin[NOWN][4];
#pragma unroll
  for (int o = 0; o < NOWN; ++o) {
    if (o > 0) __syncthreads();
#pragma unroll
    for (int j = 0; j < NG; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) red[warp][j * 4 + e][lane] = c[o * NG + j][e];
    __syncthreads();
    if (owner) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float sum = red[0][warp * 4 + e][lane];
        for (int w = 1; w < GV_WARPS; ++w) sum += red[w][warp * 4 + e][lane];
        fin[o][e] = sum;
      }
    }
  }
  if (owner) {
#pragma unroll
    for (int o = 0; o < NOWN; ++o) {
      const int j = o * NG + warp;
      const int r0 = 8 * j + 2 * t4;
      if (r0 < M) {
        if (f0 < N) epi.store2(rb0 + r0, f0, fin[o][0], pre[o][0]);
        if (f1 < N) epi.store2(rb0 + r0, f1, fin[o][2], pre[o][2]);
      }
      if (r0 + 1 < M) {
        if (f0 < N) epi.store2(rb0 + r0 + 1, f0, fin[o][1], pre[o][1]);
        if (f1 < N) epi.store2(rb0 + r0 + 1, f1, fin[o][3], pre[o][3]);
      }
    }
  }
  if constexpr (TLN) gv_tail_ln(epi.x, M, N, tln);  // residual epilogue: x rows are N = d wide
}

// online {max, sum exp} + top-1 (value desc, id asc) over the generable set
struct GvStat {
  float mx, sum, bv;
  int bi;
  __device__ __forceinline__ void init() {
    mx = -INFINITY;
    sum = 0.f;
    bv = -INFINITY;
    bi = 0x7fffffff;
  }
  __device__ __forceinline__ void add(float l, int v, int norm_allowed) {
    const bool ok = id_allowed(v);
    if (ok && better(l, v, bv, bi)) {
      bv = l;
      bi = v;
    }
    if (norm_allowed && !ok) return;
    if (l > mx) {
      sum = sum * ex2f((mx - l) * LOG2E) + 1.f;
      mx = l;
    } else {
      sum += ex2f((l - mx) * LOG2E);
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

// vocabulary columns per CTA (one partial per row): 8 warps x 16 columns, so
// the 250 CTAs at V = 32000 spread over every SM (the whole E is streamed from
// L2 once per step: per-SM L2 bandwidth is the limit)
constexpr int GV_VWARPS = 8;
constexpr int GV_VTILE = GV_VWARPS * 16;

// Vocabulary statistics for M <= 8 * NT rows: parts.ntiles must be cdiv(V, GV_VTILE).
// KT = 1: {max, sum, top-1} (greedy selection, Stage-II argmax); KT > 1 (beam search,
// decoding.py:113 top-(b+1)): the tile's KT best allowed (value desc, id asc) per row,
// picked by one thread per row from the 128 logits staged in shared memory.
template <int NT, bool LNA = false, int KT = 1>
__global__ void __launch_bounds__(GV_VWARPS * 32) gemv_vocab_kernel(const bf16* __restrict__ A, int lda,
                                                                const bf16* __restrict__ E, int V, int K, int M,
                                                                const int* __restrict__ M_dev, VocabParts parts,
                                                                int norm_allowed, GvLN ln) {
  __shared__ float4 ws[GV_VWARPS][8 * NT];
  __shared__ float lg[KT > 1 ? 8 * NT : 1][KT > 1 ? GV_VTILE : 1];  // KT > 1: the tile's logits per row
  __shared__ float2 lnst[LNA ? 8 * NT : 1];
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int n0 = blockIdx.x * GV_VTILE + warp * 16;
  const int nch = K / 32;
  const int nvalid = V - n0;
  const bool has = nvalid > 0;
  // E is the fragment-native copy (rows past V zero); CTAs past V read group 0
  const bf16* wf = gv_frag_group(E, has ? n0 : 0, K) + lane * 8;
  // first batch of weight fragments before the grid-dependency wait
  const uint64_t pol = gv_policy();
  uint4 u0[GV_MAXC], u1[GV_MAXC];
#pragma unroll
  for (int i = 0; i < GV_MAXC; ++i) {
    const int ch = min(i, nch - 1);
    u0[i] = gv_ldw(wf + (size_t)(2 * ch) * 256, pol);
    u1[i] = gv_ldw(wf + (size_t)(2 * ch + 1) * 256, pol);
  }
  pdl_wait();
  // NT = 1: the first batch of activation fragments is requested before the
  // device row count resolves (row clamped to the launch's host bound)
  constexpr bool HOIST = NT == 1 && !LNA;
  uint4 a0[HOIST ? GV_MAXC : 1];
  if constexpr (HOIST) {
    const bf16* ar = A + (size_t)min(g, M - 1) * lda + t4 * 8;
#pragma unroll
    for (int i = 0; i < GV_MAXC; ++i) a0[i] = *reinterpret_cast<const uint4*>(ar + 32 * min(i, nch - 1));
  }
  if (M_dev) M = *M_dev;
  if (M <= 0) return;  // every Stage-I row finished (uniform across the CTA)
  if (LNA) {
    gv_ln_stats(ln, M, K, lnst);
    __syncthreads();
  }
  float c[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f;
  // rolling prefetch: slot i is refilled with chunk cb + GV_MAXC + i as soon as
  // chunk cb + i is consumed, so GV_MAXC chunks stay in flight per lane
  for (int cb = 0; cb < nch; cb += GV_MAXC) {
#pragma unroll
    for (int i = 0; i < GV_MAXC; ++i) {
      if (cb + i < nch) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int r = min(8 * j + g, M - 1);
          uint4 v;
          if constexpr (HOIST) {
            v = cb == 0 ? a0[i] : gv_afrag<LNA>(A, lda, ln, lnst, K, r, 32 * (cb + i) + t4 * 8);
          } else {
            v = gv_afrag<LNA>(A, lda, ln, lnst, K, r, 32 * (cb + i) + t4 * 8);
          }
          gv_mma(c[j], u0[i].x, u1[i].x, u0[i].y, u1[i].y, v.x, v.y);
          gv_mma(c[j], u0[i].z, u1[i].z, u0[i].w, u1[i].w, v.z, v.w);
        }
        if (cb + GV_MAXC + i < nch) {
          u0[i] = gv_ldw(wf + (size_t)(2 * (cb + GV_MAXC + i)) * 256, pol);
          u1[i] = gv_ldw(wf + (size_t)(2 * (cb + GV_MAXC + i) + 1) * 256, pol);
        }
      }
    }
  }
  // per-row statistics of this warp's 16 columns, merged over the 8 lanes sharing the rows
  const int f0 = n0 + g, f1 = f0 + 8;
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      GvStat s;
      s.init();
      if (has && f0 < V) s.add(c[j][e], f0, norm_allowed);
      if (has && f1 < V) s.add(c[j][2 + e], f1, norm_allowed);
      const int row = 8 * j + 2 * t4 + e;
      if (f0 == EOS_ID && row < M) parts.eos[row] = c[j][e];
      if constexpr (KT > 1) {
        lg[row][warp * 16 + g] = c[j][e];
        lg[row][warp * 16 + g + 8] = c[j][2 + e];
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, s.mx, o);
        const float os = __shfl_xor_sync(0xffffffffu, s.sum, o);
        const float ov = __shfl_xor_sync(0xffffffffu, s.bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, s.bi, o);
        s.merge(om, os, ov, oi);
      }
      if (g == 0) ws[warp][8 * j + 2 * t4 + e] = make_float4(s.mx, s.sum, s.bv, __int_as_float(s.bi));
    }
  __syncthreads();
  if ((int)threadIdx.x < M) {
    const int r = threadIdx.x;
    GvStat s;
    s.init();
#pragma unroll 4
    for (int w = 0; w < GV_VWARPS; ++w) {
      const float4 v = ws[w][r];
      s.merge(v.x, v.y, v.z, __float_as_int(v.w));
    }
    const size_t o = (size_t)r * parts.ntiles + blockIdx.x;
    parts.mx[o] = s.mx;
    parts.sum[o] = s.sum;
    if constexpr (KT == 1) {
      parts.val[o] = s.bv;
      parts.id[o] = s.bi;
    } else {
      float tv[KT];
      int ti[KT];
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        tv[i] = -INFINITY;
        ti[i] = 0x7fffffff;
      }
      const int c0 = blockIdx.x * GV_VTILE;
      for (int q = 0; q < GV_VTILE; ++q) {
        const int id = c0 + q;
        if (id >= V || !id_allowed(id)) continue;
        float v = lg[r][q];
        int vi = id;
        if (!better(v, vi, tv[KT - 1], ti[KT - 1])) continue;
#pragma unroll
        for (int i = 0; i < KT; ++i)  // insertion into the sorted list
          if (better(v, vi, tv[i], ti[i])) {
            const float sv = tv[i];
            const int si = ti[i];
            tv[i] = v;
            ti[i] = vi;
            v = sv;
            vi = si;
          }
      }
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        parts.val[o * KT + i] = tv[i];
        parts.id[o * KT + i] = ti[i];
      }
    }
  }
}

}  // namespace hrt
