// Stage-I decoder layers for a handful of live rows (greedy, R <= 4) as ONE
// kernel on one 16-CTA thread-block cluster (infer.py:234-291 up to the final
// LayerNorm; the vocabulary projection and the selection stay separate).
//
// At batch 1 a decoder step is a chain of ~11 dependent kernels whose
// individual work is tiny (the layer's 7.3 MB of bf16 weights are L2
// resident); the step time is the sum of their dependent latencies. Here the
// chain lives inside one cluster:
//   * every CTA owns a slice of each projection's output features (QKV by
//     head halves, so a head's q / k / v live on a CTA pair); its weight rows
//     stream into a 4-slot shared-memory ring with 1-D bulk copies
//     (cp.async.bulk, mbarrier completion), issued ahead -- the first slots
//     before the grid-dependency wait (weights never depend on the previous
//     kernel);
//   * activations are replicated in every CTA (x fp32, y / ctx / hidden bf16:
//     the same operand precisions as the unfused path); a CTA computes its
//     slice and writes it into every CTA's shared memory (DSMEM), and one
//     cluster barrier (hardware, release / acquire) publishes it;
//   * attention: the CTA pair of head h splits the keys, each produces an
//     online-softmax partial (max, sum, o[64]) that it broadcasts; every CTA
//     merges the two partials of all heads itself (no second exchange);
//   * LayerNorms are recomputed redundantly per CTA from the replicated x.
// 8 cluster barriers per decoder layer replace 10 kernel boundaries.
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace hrt {

constexpr int DC_CN = 16;  // CTAs per cluster (non-portable size)
constexpr int DC_THREADS = 256;
constexpr int DC_D = 512, DC_FF = 2048, DC_H = 8, DC_DH = 64;
constexpr int DC_RMAX = 4;
constexpr int DC_CHUNK = 32 * 1024;  // bytes per weight chunk (one ring slot)
constexpr int DC_CPL = 14;  // chunks per layer: q k v | wo | qc | woc | w1 x4 | w2 x4
constexpr int DC_MAXL = 2;  // decoder layers whose biases / LN parameters are staged in shared memory
constexpr int DC_PRM = 352 + 6 * DC_D;  // floats per layer: own bias slices + six LayerNorm vectors

struct DcLayer {
  const bf16 *wqkv, *wo, *wqc, *woc, *w1, *w2;
  const float *bqkv, *bo, *bqc, *boc, *b1, *b2, *ln2g, *ln2b, *ln3g, *ln3b, *ln1g_next, *ln1b_next;
};
struct DcParams {
  DcLayer L[DC_MAXL];
  int Ld;
  const bf16* xkv;  // [tokens][Ld * 2 D] cross K / V (layer i: K at 2 i D, V at (2 i + 1) D)
  int xstride;
  const int* src_off;  // [rows] first memory token of the row's sentence
  const int* src_len;
  bf16* kc;  // [Ld][rcap][cap][D] self-attention cache
  bf16* vc;
  int cap, rcap;
  float* x;  // [R][D] residual stream (embedding on entry)
  bf16* y;   // [R][D] LN1(x) on entry; the final LayerNorm on exit
  const StepCtl* ctl;
  int R_host, t_host;
  float att_scale;
  int dbg;  // timing attribution only (wrong results): 1 no weight copies, 2 no attention, 4 no broadcasts
};

// smem layout (bytes) for row bucket RB: the ring takes what the row buffers leave (five
// 32 KB slots for single-row buckets, four otherwise)
template <int RB>
struct DcSmem {
  static constexpr int NSLOT = RB == 1 ? 5 : 4;
  static constexpr int RING = 0;
  static constexpr int XS = RING + NSLOT * DC_CHUNK;          // float [R][D]
  static constexpr int YS = XS + RB * DC_D * 4;              // bf16 [R][D]   (LN output, GEMV input)
  static constexpr int CS = YS + RB * DC_D * 2;              // bf16 [R][D]   (attention context)
  static constexpr int HS = CS + RB * DC_D * 2;              // bf16 [R][FF]  (FFN hidden)
  static constexpr int QS = HS + RB * DC_FF * 2;             // float [R][3][64] (this head's q / k / v)
  static constexpr int PS = QS + RB * 3 * 64 * 4;            // float [R][H][2][68] (attention partials)
  static constexpr int OS = PS + RB * DC_H * 2 * 68 * 4;     // float [R][128] GEMV slice staging
  static constexpr int WS = OS + RB * 128 * 4;               // float [8 warps][68] attention merge
  static constexpr int PRM = WS + 8 * 68 * 4;                // float [MAXL][DC_PRM] static parameters
  static constexpr int BAR = PRM + DC_MAXL * DC_PRM * 4;
  static constexpr int TOTAL = BAR + 64 + 128;
  static_assert(TOTAL <= 227 * 1024, "decode cluster shared memory");
};

__device__ __forceinline__ unsigned long long dc_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void dc_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint32_t dc_mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void dc_st4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// global source of chunk j of layer l for CTA c (32 KB of contiguous weight rows)
__device__ __forceinline__ const bf16* dc_chunk_src(const DcLayer& w, int j, int c) {
  const int hh = c >> 1, half = c & 1, qrow = hh * 64 + half * 32;
  switch (j) {
    case 0: return w.wqkv + (size_t)qrow * DC_D;
    case 1: return w.wqkv + (size_t)(DC_D + qrow) * DC_D;
    case 2: return w.wqkv + (size_t)(2 * DC_D + qrow) * DC_D;
    case 3: return w.wo + (size_t)(32 * c) * DC_D;
    case 4: return w.wqc + (size_t)(32 * c) * DC_D;
    case 5: return w.woc + (size_t)(32 * c) * DC_D;
    case 6: case 7: case 8: case 9: return w.w1 + (size_t)(128 * c + 32 * (j - 6)) * DC_D;
    default: return w.w2 + (size_t)(32 * c + 8 * (j - 10)) * DC_FF;
  }
}

// GEMV over a chunk in shared memory: out[r][f] = sum_k W[f][k] in[r][k] for
// NF rows f of the chunk (row length K), R input rows (bf16, row stride K).
// Warp w takes rows f = w, w + 8, ...; lanes split K in 16-byte groups.
template <int K, int NF, int R, int LDO = NF>
__device__ __forceinline__ void dc_gemv(const bf16* __restrict__ W, const bf16* __restrict__ in,
                                        float* __restrict__ out /* [R][LDO], columns 0..NF-1 */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int FPW = NF / 8;  // rows per warp
  float acc[FPW][R];
#pragma unroll
  for (int i = 0; i < FPW; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[i][r] = 0.f;
#pragma unroll
  for (int it = 0; it < K / 256; ++it) {
    const int k0 = (it * 32 + lane) * 8;
    float a[R][8];
#pragma unroll
    for (int r = 0; r < R; ++r) load8(in + (size_t)r * K + k0, a[r]);
#pragma unroll
    for (int i = 0; i < FPW; ++i) {
      float wv[8];
      load8(W + (size_t)(warp + 8 * i) * K + k0, wv);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[i][r] = fmaf(wv[e], a[r][e], acc[i][r]);
    }
  }
#pragma unroll
  for (int i = 0; i < FPW; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float s = warp_sum(acc[i][r]);  // unconditional: no divergent shuffles
      if (lane == 0) out[r * LDO + warp + 8 * i] = s;
    }
}

// LayerNorm of R fp32 rows of D into bf16 (warp per row, kernels.py:42-57)
// (every warp normalises row warp % R; warps < R store: no divergent shuffles)
template <int R>
__device__ __forceinline__ void dc_layernorm(const float* __restrict__ xs, const float* __restrict__ g,
                                             const float* __restrict__ b, bf16* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const int r = warp % R;
    const float* xr = xs + r * DC_D;
    float v[16];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 q = *reinterpret_cast<const float4*>(xr + (lane + 32 * i) * 4);
      v[4 * i] = q.x;
      v[4 * i + 1] = q.y;
      v[4 * i + 2] = q.z;
      v[4 * i + 3] = q.w;
      s += (q.x + q.y) + (q.z + q.w);
    }
    const float mean = warp_sum(s) / DC_D;
    float q2 = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float a = v[i] - mean;
      q2 += a * a;
    }
    const float inv = 1.0f / sqrtf(warp_sum(q2) / DC_D + 1e-5f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c4 = (lane + 32 * i) * 4;
      const float4 gg = *reinterpret_cast<const float4*>(g + c4);
      const float4 bb = *reinterpret_cast<const float4*>(b + c4);
      __nv_bfloat162 lo = __floats2bfloat162_rn((v[4 * i] - mean) * inv * gg.x + bb.x,
                                                (v[4 * i + 1] - mean) * inv * gg.y + bb.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn((v[4 * i + 2] - mean) * inv * gg.z + bb.z,
                                                (v[4 * i + 3] - mean) * inv * gg.w + bb.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      if (warp < R) *reinterpret_cast<uint2*>(out + r * DC_D + c4) = u;
    }
  }
}

// One head-half of single-query attention: keys j in [j0, j1) (key rows of
// 64 bf16 at kbase + j * kstride / vbase + ...; key `jnew`, if in range, is the
// fp32 new key / value in smem instead), query q (fp32 smem, pre-scaled).
// Leaves the CTA's (max, sum, o[64]) partial in part[0..65].
__device__ __forceinline__ void dc_attend(const float* __restrict__ q, const bf16* __restrict__ kbase,
                                          const bf16* __restrict__ vbase, size_t kstride, int j0, int j1, int jnew,
                                          const float* __restrict__ knew, const float* __restrict__ vnew,
                                          float* __restrict__ wbuf /* [8][68] */, float* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float q0 = q[2 * lane], q1 = q[2 * lane + 1];
  float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f;
  // keys j0 + 64 b + warp + 8 u: up to 8 per warp per block, all loads issued before any use;
  // the block count is CTA-uniform and every shuffle runs unconditionally
  const int nblk = (j1 - j0 + 63) / 64;
  for (int bk = 0; bk < nblk; ++bk) {
    const int jb = j0 + bk * 64 + warp;
    const int nu = min(8, (j1 - j0 - bk * 64 + 7) / 8);  // key slots in use (CTA-uniform)
    __nv_bfloat162 kk[8], vv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = jb + 8 * u;
      if (j < j1 && j != jnew) {
        kk[u] = *reinterpret_cast<const __nv_bfloat162*>(kbase + j * kstride + 2 * lane);
        vv[u] = *reinterpret_cast<const __nv_bfloat162*>(vbase + j * kstride + 2 * lane);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u >= nu) break;
      const int j = jb + 8 * u;
      const bool valid = j < j1;
      float k0 = 0.f, k1 = 0.f, v0 = 0.f, v1 = 0.f;
      if (j == jnew) {
        k0 = knew[2 * lane];
        k1 = knew[2 * lane + 1];
        v0 = vnew[2 * lane];
        v1 = vnew[2 * lane + 1];
      } else if (valid) {
        const float2 kf = __bfloat1622float2(kk[u]), vf = __bfloat1622float2(vv[u]);
        k0 = kf.x;
        k1 = kf.y;
        v0 = vf.x;
        v1 = vf.y;
      }
      const float sc = warp_sum(q0 * k0 + q1 * k1);
      if (valid) {
        const float mn = fmaxf(m, sc);
        const float cc = ex2f((m - mn) * LOG2E);
        const float pp = ex2f((sc - mn) * LOG2E);
        l = l * cc + pp;
        o0 = o0 * cc + pp * v0;
        o1 = o1 * cc + pp * v1;
        m = mn;
      }
    }
  }
  float* wb = wbuf + warp * 68;
  if (lane == 0) {
    wb[0] = m;
    wb[1] = l;
  }
  wb[2 + 2 * lane] = o0;
  wb[3 + 2 * lane] = o1;
  __syncthreads();
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 8; ++w) M = fmaxf(M, wbuf[w * 68]);
    float L = 0.f, a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const float mw = wbuf[w * 68];
      const float c = mw == -INFINITY ? 0.f : ex2f((mw - M) * LOG2E);
      L += wbuf[w * 68 + 1] * c;
      a0 += wbuf[w * 68 + 2 + 2 * lane] * c;
      a1 += wbuf[w * 68 + 3 + 2 * lane] * c;
    }
    if (lane == 0) {
      part[0] = M;
      part[1] = L;
    }
    part[2 + 2 * lane] = a0;
    part[3 + 2 * lane] = a1;
  }
  __syncthreads();
}

// merge the two halves' partials of every head into ctx (bf16 [D]) for one row
__device__ __forceinline__ void dc_merge_heads(const float* __restrict__ prow /* [H][2][68] */,
                                               bf16* __restrict__ ctx) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp = head
  const float* a = prow + warp * 2 * 68;
  const float* b = a + 68;
  const float M = fmaxf(a[0], b[0]);
  const float ca = a[0] == -INFINITY ? 0.f : ex2f((a[0] - M) * LOG2E);
  const float cb = b[0] == -INFINITY ? 0.f : ex2f((b[0] - M) * LOG2E);
  const float inv = 1.0f / (a[1] * ca + b[1] * cb);
  const float o0 = (a[2 + 2 * lane] * ca + b[2 + 2 * lane] * cb) * inv;
  const float o1 = (a[3 + 2 * lane] * ca + b[3 + 2 * lane] * cb) * inv;
  *reinterpret_cast<__nv_bfloat162*>(ctx + warp * 64 + 2 * lane) = __floats2bfloat162_rn(o0, o1);
}

// RB: the launch's row bucket (1, 2 or 4); rows past the live count are computed and
// discarded (their buffers exist), so every loop and shuffle is compile-time uniform
template <int RB>
__global__ void __cluster_dims__(DC_CN, 1, 1) __launch_bounds__(DC_THREADS, 1) decode_cluster_kernel(DcParams p) {
  using SM = DcSmem<RB>;
  constexpr int DC_NSLOT = SM::NSLOT;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* ring = dsm + SM::RING;
  float* xs = reinterpret_cast<float*>(dsm + SM::XS);
  bf16* ys = reinterpret_cast<bf16*>(dsm + SM::YS);
  bf16* cs = reinterpret_cast<bf16*>(dsm + SM::CS);
  bf16* hs = reinterpret_cast<bf16*>(dsm + SM::HS);
  float* qs = reinterpret_cast<float*>(dsm + SM::QS);
  float* ps = reinterpret_cast<float*>(dsm + SM::PS);
  float* os = reinterpret_cast<float*>(dsm + SM::OS);
  float* wsb = reinterpret_cast<float*>(dsm + SM::WS);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + SM::BAR);  // [DC_NSLOT]
  float* prm = reinterpret_cast<float*>(dsm + SM::PRM);

  pdl_trigger();
  unsigned long long ts[40];
  int nts = 0;
  const bool trace = (p.dbg & 8) != 0;
#define DC_TS() if (trace) ts[nts++] = dc_now()
  DC_TS();
  // the grid is exactly one cluster, so the CTA rank is blockIdx.x -- which the compiler
  // knows to be uniform (loops bounded by it keep their shuffles non-divergent)
  const int c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = c >> 1, half = c & 1;
  const int nchunks = p.Ld * DC_CPL;
  if (tid == 0) {
    for (int s = 0; s < DC_NSLOT; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // weight ring: chunk i lives in slot i % NSLOT; issued = chunks requested so far
  int issued = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  auto issue_upto = [&](int n) {
    n = min(n, nchunks);
    if (tid == 0 && !(p.dbg & 1))  // (dbg 1: no weight copies at all, stale ring contents)
      for (int i = issued; i < n; ++i) {
        uint64_t* bar = &full[i % DC_NSLOT];
        mbar_arrive_expect_tx(bar, DC_CHUNK);
        dc_bulk_load(ring + (i % DC_NSLOT) * DC_CHUNK, dc_chunk_src(p.L[i / DC_CPL], i % DC_CPL, c), DC_CHUNK, bar,
                     pol);
      }
    issued = max(issued, n);
  };
  auto chunk = [&](int i) -> const bf16* {
    if (!(p.dbg & 1)) mbar_wait(&full[i % DC_NSLOT], (i / DC_NSLOT) & 1);
    return reinterpret_cast<const bf16*>(ring + (i % DC_NSLOT) * DC_CHUNK);
  };
  issue_upto(DC_NSLOT);  // weights do not depend on the previous kernel
  // static parameters of every layer into shared memory: this CTA's bias slices and
  // the LayerNorm vectors (also independent of the previous kernel)
  // (float4 items: 24 bias slices of 4, then the six LayerNorm vectors; every load is
  // issued before any store so the requests overlap)
  for (int li = 0; li < p.Ld; ++li) {
    const DcLayer& w = p.L[li];
    float4* pr4 = reinterpret_cast<float4*>(prm + li * DC_PRM);
    const int qrow = hh * 64 + half * 32;
    constexpr int N4 = DC_PRM / 4, PER = (N4 + DC_THREADS - 1) / DC_THREADS;
    float4 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = tid + k * DC_THREADS;
      const float* src = nullptr;
      if (i < 24) src = w.bqkv + (i >> 3) * DC_D + qrow + 4 * (i & 7);
      else if (i < 32) src = w.bo + 32 * c + 4 * (i - 24);
      else if (i < 40) src = w.bqc + 32 * c + 4 * (i - 32);
      else if (i < 48) src = w.boc + 32 * c + 4 * (i - 40);
      else if (i < 80) src = w.b1 + 128 * c + 4 * (i - 48);
      else if (i < 88) src = w.b2 + 32 * c + 4 * (i - 80);
      else if (i < N4) {
        const int q = i - 88, vec = q / (DC_D / 4), e = 4 * (q - vec * (DC_D / 4));
        src = (vec == 0 ? w.ln2g : vec == 1 ? w.ln2b : vec == 2 ? w.ln3g : vec == 3 ? w.ln3b
                         : vec == 4 ? w.ln1g_next : w.ln1b_next) + e;
      }
      v[k] = src ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (tid + k * DC_THREADS < N4) pr4[tid + k * DC_THREADS] = v[k];
  }
  pdl_wait();
  DC_TS();
  // the live rows' x / y are requested before the device row count resolves (rows up to
  // the launch's host bound, which the buffers always hold)
  for (int i = tid; i < RB * DC_D / 4; i += DC_THREADS)
    reinterpret_cast<float4*>(xs)[i] = reinterpret_cast<const float4*>(p.x)[i];
  for (int i = tid; i < RB * DC_D / 8; i += DC_THREADS)
    reinterpret_cast<uint4*>(ys)[i] = reinterpret_cast<const uint4*>(p.y)[i];
  int Rlive = p.R_host, t = p.t_host;
  if (p.ctl) {
    Rlive = p.ctl->R;
    t = p.ctl->t;
  }
  if (Rlive <= 0) {  // every row finished: drain the ring before leaving
    if (tid == 0 && !(p.dbg & 1))
      for (int i = 0; i < issued; ++i) mbar_wait(&full[i % DC_NSLOT], (i / DC_NSLOT) & 1);
    cluster_sync_all();
    return;
  }
  constexpr int R = RB;
  __syncthreads();
  DC_TS();

  // broadcast nf fp32 values per row from os into every CTA's dst (fp32 [R][ld] at col0),
  // or (bf16) into a bf16 array; 16 threads per destination CTA
  auto bcast_f32 = [&](float* dst, int ld, int col0, int nf) {
    if (p.dbg & 4) return;
    const int per = nf / 4;  // float4 per row
    for (int idx = tid; idx < DC_CN * R * per; idx += DC_THREADS) {
      const int dstc = idx / (R * per), rem = idx - dstc * (R * per), r = rem / per, q4 = rem - r * per;
      const float4 v = reinterpret_cast<const float4*>(os + r * nf)[q4];
      uint4 u = make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w));
      dc_st4(dc_mapa(dst + r * ld + col0 + 4 * q4, (uint32_t)dstc), u);
    }
  };
  auto bcast_bf16 = [&](bf16* dst, int ld, int col0, int nf) {
    if (p.dbg & 4) return;
    const int per = nf / 8;  // 8 bf16 per 16-byte store
    for (int idx = tid; idx < DC_CN * R * per; idx += DC_THREADS) {
      const int dstc = idx / (R * per), rem = idx - dstc * (R * per), r = rem / per, q8 = rem - r * per;
      const float* sv = os + r * nf + 8 * q8;
      uint4 u;
      uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(sv[2 * e], sv[2 * e + 1]);
        w[e] = *reinterpret_cast<uint32_t*>(&b2);
      }
      dc_st4(dc_mapa(dst + r * ld + col0 + 8 * q8, (uint32_t)dstc), u);
    }
  };

  for (int li = 0; li < p.Ld; ++li) {
    const float* pr = prm + li * DC_PRM;
    const float *ln2g = pr + 352, *ln2b = ln2g + DC_D, *ln3g = ln2b + DC_D, *ln3b = ln3g + DC_D,
                *lnng = ln3b + DC_D, *lnnb = lnng + DC_D;
    const int cb = li * DC_CPL;
    bf16* kc = p.kc + (size_t)li * p.rcap * p.cap * DC_D;
    bf16* vc = p.vc + (size_t)li * p.rcap * p.cap * DC_D;
    // ---- self-attention projections: q / k / v of head hh, dims half * 32 .. +32 ----
    dc_gemv<DC_D, 32, R, 96>(chunk(cb), ys, os);
    DC_TS();
    dc_gemv<DC_D, 32, R, 96>(chunk(cb + 1), ys, os + 32);
    dc_gemv<DC_D, 32, R, 96>(chunk(cb + 2), ys, os + 64);
    __syncthreads();
    DC_TS();
    issue_upto(cb + 3 + DC_NSLOT);  // a slot is refilled as soon as every warp has consumed it
    {
      for (int idx = tid; idx < R * 96; idx += DC_THREADS) {
        const int r = idx / 96, jf = idx - r * 96, j = jf >> 5, f = jf & 31;
        float v = os[r * 96 + jf] + pr[jf];
        if (j == 0) v *= p.att_scale;
        else v = __bfloat162float(__float2bfloat16_rn(v));  // the cache holds bf16 k / v
        // own copy and the partner CTA's (the head's other half)
        qs[(r * 3 + j) * 64 + half * 32 + f] = v;
        const uint32_t a = dc_mapa(qs + (r * 3 + j) * 64 + half * 32 + f, (uint32_t)(c ^ 1));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
      }
    }
    DC_TS();
    cluster_sync_all();  // B1: the pair's q / k / v complete
    DC_TS();
    // the new key / value into the cache after B1 (global stores before a release barrier would
    // hold it up; this step's attention takes slot t from shared memory, later steps from here)
    for (int idx = tid; idx < R * 64; idx += DC_THREADS) {
      const int r = idx >> 6, j = 1 + (idx >> 5 & 1), f = idx & 31;
      bf16* dst = j == 1 ? kc : vc;
      dst[((size_t)r * p.cap + t) * DC_D + hh * 64 + half * 32 + f] =
          __float2bfloat16_rn(qs[(r * 3 + j) * 64 + half * 32 + f]);
    }
    // ---- self-attention over slots 0..t: the pair splits the keys ----
    for (int r = 0; r < ((p.dbg & 2) ? 0 : R); ++r) {
      const int nk = t + 1, mid = (nk + 1) / 2;
      const int j0 = half ? mid : 0, j1 = half ? nk : mid;
      const size_t rb = (size_t)r * p.cap * DC_D + hh * 64;
      float* part = os;  // [68] staging
      dc_attend(qs + (r * 3) * 64, kc + rb, vc + rb, DC_D, j0, j1, t, qs + (r * 3 + 1) * 64, qs + (r * 3 + 2) * 64,
                wsb, part);
      // broadcast the partial to every CTA: ps[r][hh][half][0..65]
      for (int idx = tid; idx < DC_CN * 17; idx += DC_THREADS) {
        const int dstc = idx / 17, q4 = idx - dstc * 17;
        const float4 v = reinterpret_cast<const float4*>(part)[q4];
        dc_st4(dc_mapa(ps + ((r * DC_H + hh) * 2 + half) * 68 + 4 * q4, (uint32_t)dstc),
               make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)));
      }
      __syncthreads();
    }
    cluster_sync_all();  // B2: every head's partials everywhere
    DC_TS();
    for (int r = 0; r < R; ++r) dc_merge_heads(ps + r * DC_H * 2 * 68, cs + r * DC_D);
    __syncthreads();
    // ---- Wo + residual: x[32 c .. +32] ----
    dc_gemv<DC_D, 32, R>(chunk(cb + 3), cs, os);
    __syncthreads();
    issue_upto(cb + 4 + DC_NSLOT);
    for (int idx = tid; idx < R * 32; idx += DC_THREADS) {
      const int r = idx >> 5, f = idx & 31, col = 32 * c + f;
      os[r * 32 + f] = xs[r * DC_D + col] + (os[r * 32 + f] + pr[96 + f]);
    }
    __syncthreads();
    bcast_f32(xs, DC_D, 32 * c, 32);
    cluster_sync_all();  // B3
    DC_TS();
    dc_layernorm<R>(xs, ln2g, ln2b, ys);
    __syncthreads();
    // ---- cross-attention query: dims 32 c .. +32 = head hh, half ----
    dc_gemv<DC_D, 32, R>(chunk(cb + 4), ys, os);
    __syncthreads();
    issue_upto(cb + 5 + DC_NSLOT);
    for (int idx = tid; idx < R * 32; idx += DC_THREADS) {
      const int r = idx >> 5, f = idx & 31;
      const float v = (os[r * 32 + f] + pr[128 + f]) * p.att_scale;
      qs[(r * 3) * 64 + half * 32 + f] = v;
      const uint32_t a = dc_mapa(qs + (r * 3) * 64 + half * 32 + f, (uint32_t)(c ^ 1));
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
    }
    cluster_sync_all();  // B4
    DC_TS();
    // ---- cross-attention over the sentence memory ----
    for (int r = 0; r < ((p.dbg & 2) ? 0 : R); ++r) {
      const int S = p.src_len[r], mid = (S + 1) / 2;
      const int j0 = half ? mid : 0, j1 = half ? S : mid;
      const bf16* kb = p.xkv + (size_t)p.src_off[r] * p.xstride + 2 * li * DC_D + hh * 64;
      float* part = os;
      dc_attend(qs + (r * 3) * 64, kb, kb + DC_D, p.xstride, j0, j1, -1, nullptr, nullptr, wsb, part);
      for (int idx = tid; idx < DC_CN * 17; idx += DC_THREADS) {
        const int dstc = idx / 17, q4 = idx - dstc * 17;
        const float4 v = reinterpret_cast<const float4*>(part)[q4];
        dc_st4(dc_mapa(ps + ((r * DC_H + hh) * 2 + half) * 68 + 4 * q4, (uint32_t)dstc),
               make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w)));
      }
      __syncthreads();
    }
    cluster_sync_all();  // B5
    DC_TS();
    for (int r = 0; r < R; ++r) dc_merge_heads(ps + r * DC_H * 2 * 68, cs + r * DC_D);
    __syncthreads();
    // ---- Woc + residual ----
    dc_gemv<DC_D, 32, R>(chunk(cb + 5), cs, os);
    __syncthreads();
    issue_upto(cb + 6 + DC_NSLOT);
    for (int idx = tid; idx < R * 32; idx += DC_THREADS) {
      const int r = idx >> 5, f = idx & 31, col = 32 * c + f;
      os[r * 32 + f] = xs[r * DC_D + col] + (os[r * 32 + f] + pr[160 + f]);
    }
    __syncthreads();
    bcast_f32(xs, DC_D, 32 * c, 32);
    cluster_sync_all();  // B6
    DC_TS();
    dc_layernorm<R>(xs, ln3g, ln3b, ys);
    __syncthreads();
    // ---- W1 + ReLU: hidden[128 c .. +128] (four 32-row chunks) ----
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      dc_gemv<DC_D, 32, R, 128>(chunk(cb + 6 + j), ys, os + 32 * j);
      __syncthreads();
      issue_upto(cb + 7 + j + DC_NSLOT);  // the W2 chunks stream in under W1
    }
    for (int idx = tid; idx < R * 128; idx += DC_THREADS) os[idx] = fmaxf(os[idx] + pr[192 + (idx & 127)], 0.f);
    __syncthreads();
    bcast_bf16(hs, DC_FF, 128 * c, 128);
    cluster_sync_all();  // B7
    DC_TS();
    // ---- W2 + residual: x[32 c .. +32] over K = FF (four 8-row chunks) ----
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const bf16* wch = chunk(cb + 10 + j);
      DC_TS();
      dc_gemv<DC_FF, 8, R, 32>(wch, hs, wsb + 8 * j);
      __syncthreads();
      issue_upto(cb + 11 + j + DC_NSLOT);  // the next layer's chunks
    }
    DC_TS();
    for (int idx = tid; idx < R * 32; idx += DC_THREADS) {
      const int r = idx >> 5, f = idx & 31, col = 32 * c + f;
      os[r * 32 + f] = xs[r * DC_D + col] + (wsb[r * 32 + f] + pr[320 + f]);
    }
    __syncthreads();
    bcast_f32(xs, DC_D, 32 * c, 32);
    cluster_sync_all();  // B8
    DC_TS();
    // next layer's LN1, or the final LayerNorm into the vocabulary operand
    dc_layernorm<R>(xs, lnng, lnnb, ys);
    __syncthreads();
  }
  // final LN output: CTA c writes columns 32 c .. +32 of every row
  for (int idx = tid; idx < R * 4; idx += DC_THREADS) {
    const int r = idx >> 2, q8 = idx & 3;
    *reinterpret_cast<uint4*>(p.y + (size_t)r * DC_D + 32 * c + 8 * q8) =
        *reinterpret_cast<const uint4*>(ys + r * DC_D + 32 * c + 8 * q8);
  }
  // (no closing cluster barrier: the last remote shared-memory writes were published by B8)
  DC_TS();
  if (trace && c == 0 && tid == 0 && t == 5) {
    printf("dc trace t=%d R=%d:", t, R);
    for (int i = 1; i < nts; ++i) printf(" %.2f", (ts[i] - ts[i - 1]) * 1e-3);
    printf("  total %.2f us\n", (ts[nts - 1] - ts[0]) * 1e-3);
  }
#undef DC_TS
}

}  // namespace hrt
