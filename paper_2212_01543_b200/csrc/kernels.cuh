// Non-GEMM kernels of the HRT inference path (sm_100a).
//
// Every kernel cites the reference operation it implements
// (/root/reference/pkg/src/hrt/...). Residual streams are fp32; matrix
// operands (T) are fp32 or bf16; all reductions accumulate in fp32, and
// search scores in fp64 as the reference's Python floats do.
#pragma once
#include <type_traits>
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
                                const int* __restrict__ pos_dev, const int* __restrict__ M_dev, int M, int d,
                                float scale, const T* __restrict__ E, const float* __restrict__ pe,
                                const float* __restrict__ g, const float* __restrict__ b, float* __restrict__ x,
                                T* __restrict__ y);

// ---------------------------------------------------------------------------
// Vectorised LayerNorm for d % 128 == 0: each lane owns NV float4 chunks of
// the row (16-byte loads, NV independent loads in flight per lane).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void store4v(T* p, float4 v);
template <>
__device__ __forceinline__ void store4v<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
template <>
__device__ __forceinline__ void store4v<bf16>(bf16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

template <typename T, int NV>
__global__ void layernorm_vec_kernel(const float* __restrict__ x, const int* __restrict__ M_dev, int M, int d,
                                     const float* __restrict__ g, const float* __restrict__ b, T* __restrict__ y,
                                     const int* __restrict__ out_row, float* __restrict__ y32) {
  pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  float4 v[NV], gv[NV], bv[NV];
  // gain / bias never change: requested before the grid-dependency wait
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    gv[i] = __ldg(reinterpret_cast<const float4*>(g) + lane + 32 * i);
    bv[i] = __ldg(reinterpret_cast<const float4*>(b) + lane + 32 * i);
  }
  pdl_wait();
  // the row is requested before the device row count resolves (clamped to the
  // launch's host bound, which the buffer always holds)
  {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)min(row, M - 1) * d);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = xr[lane + 32 * i];
  }
  if (M_dev) M = *M_dev;
  if (row >= M) return;
  const int orow = out_row ? out_row[row] : row;
  if (orow < 0) return;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a = v[i].x - mean, bb = v[i].y - mean, c = v[i].z - mean, e = v[i].w - mean;
    q += (a * a + bb * bb) + (c * c + e * e);
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = (lane + 32 * i) * 4;
    const float4 gg = gv[i], bb = bv[i];
    float4 o;
    o.x = (v[i].x - mean) * inv * gg.x + bb.x;
    o.y = (v[i].y - mean) * inv * gg.y + bb.y;
    o.z = (v[i].z - mean) * inv * gg.z + bb.z;
    o.w = (v[i].w - mean) * inv * gg.w + bb.w;
    store4v<T>(y + (size_t)orow * d + c4, o);
    if (y32) store4v<float>(y32 + (size_t)orow * d + c4, o);
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
  pdl_enter();
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

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float LOG2E = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// vector helpers: load 8 consecutive T as fp32
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load8(const float* p, float* o) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void load8(const bf16* p, float* o) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
}

__device__ __forceinline__ void loadvec(const float* p, float* o) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
}
__device__ __forceinline__ void loadvec(const bf16* p, float* o) { load8(p, o); }

// ---------------------------------------------------------------------------
// Ragged ("varlen") multi-head attention for whole sequences:
//   encoder self-attention            infer.py:196-203   (full)
//   Stage-II self-attention           infer.py:364-373   (full or causal, key padding)
//   Stage-II cross-attention          infer.py:377-385   (keys = sentence memory)
// Sequence s owns query rows [q_off[s], q_off[s] + q_slot[s]) of which the
// first q_len[s] are real (the rest get zero output), and attends key rows
// [kv_off[kvs], kv_off[kvs] + kv_len[kvs]) with kvs = kv_map ? kv_map[s] : s.
// Keys whose key_ok byte is 0 are masked (additive -1e9 in the reference;
// exp underflows to exactly 0 either way).
// grid = (work items, heads): item i = (sequence, 32-query block), built on
// the host so no CTA is empty. Every LANE owns one query (q and the output
// accumulator in registers); the 4 warps split each 64-key shared-memory
// chunk 16 keys apiece with private online-softmax state, merged at the end.
// ---------------------------------------------------------------------------
constexpr int AP_WARPS = 4, AP_KC = 64, AP_KG = 16;

template <typename T, int DH>
__global__ void __launch_bounds__(AP_WARPS * 32) attn_prefill_kernel(
    const int2* __restrict__ items, const T* __restrict__ q, int q_stride, const T* __restrict__ k,
    const T* __restrict__ v, int kv_stride, T* __restrict__ out, int out_stride, const int* __restrict__ q_off,
    const int* __restrict__ q_slot, const int* __restrict__ q_len, const int* __restrict__ kv_map,
    const int* __restrict__ kv_off, const int* __restrict__ kv_len, const unsigned char* __restrict__ key_ok,
    int causal, float scale) {
  pdl_enter();
  __shared__ __align__(16) float Ks[AP_KC][DH];
  __shared__ __align__(16) float Vs[AP_KC][DH];
  __shared__ float kbias[AP_KC];
  __shared__ float wm[AP_WARPS][32], wl[AP_WARPS][32];
  const int2 it = items[blockIdx.x];
  const int s = it.x, qbeg = it.y * 32, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qslot = q_slot[s];
  const int qlen = q_len[s];
  const int kvs = kv_map ? kv_map[s] : s;
  const int kb = kv_off[kvs];
  const int L = kv_len[kvs];
  const int hoff = h * DH;
  const int qb = q_off[s];
  const int qi = qbeg + lane;
  const bool live = qi < qlen;
  float qr[DH], o[DH];
  if (live) {
    const T* src = q + (size_t)(qb + qi) * q_stride + hoff;
    if (DH % 8 == 0) {
#pragma unroll
      for (int c = 0; c < DH; c += 8) load8(src + c, qr + c);
    } else {
#pragma unroll
      for (int c = 0; c < DH; ++c) qr[c] = to_f(src[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < DH; ++c) {
    qr[c] = live ? qr[c] * scale : 0.f;
    o[c] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int qmax = min(qslot, qbeg + 32) - 1;
  const int Lc = causal ? min(L, qmax + 1) : L;
  const bool any_live = qbeg < qlen;
  for (int j0 = 0; j0 < Lc; j0 += AP_KC) {
    const int nk = min(AP_KC, Lc - j0);
    __syncthreads();  // previous chunk fully consumed
    constexpr int V8 = DH >= 8 ? DH / 8 : 1;
    for (int idx = threadIdx.x; idx < nk * V8; idx += blockDim.x) {
      const int j = idx / V8, c8 = (idx % V8) * 8;
      const size_t r = (size_t)(kb + j0 + j) * kv_stride + hoff + c8;
      if (DH >= 8) {
        load8(k + r, &Ks[j][c8]);
        load8(v + r, &Vs[j][c8]);
      } else {
        for (int c = 0; c < DH; ++c) {
          Ks[j][c] = to_f(k[r + c]);
          Vs[j][c] = to_f(v[r + c]);
        }
      }
    }
    for (int j = threadIdx.x; j < AP_KC; j += blockDim.x)
      kbias[j] = (j < nk && (key_ok == nullptr || key_ok[kb + j0 + j])) ? 0.f : -INFINITY;
    __syncthreads();
    const int g = warp * AP_KG;  // this warp's 16 keys of the chunk
    if (!any_live || g >= nk) continue;
    float sc[AP_KG];
    float cm = -INFINITY;
#pragma unroll
    for (int u = 0; u < AP_KG; ++u) {
      const int j = g + u;
      float a = -INFINITY;
      if (j < nk && !(causal && j0 + j > qi)) {
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < DH; c += 2) {
          a0 = fmaf(qr[c], Ks[j][c], a0);
          if (c + 1 < DH) a1 = fmaf(qr[c + 1], Ks[j][c + 1], a1);
        }
        a = a0 + a1 + kbias[j];
      }
      sc[u] = a;
      cm = fmaxf(cm, a);
    }
    const float mn = fmaxf(m, cm);
    if (mn == -INFINITY) continue;
    const float corr = ex2f((m - mn) * LOG2E);
    l *= corr;
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] *= corr;
    m = mn;
    const float ms = mn * LOG2E;
#pragma unroll
    for (int u = 0; u < AP_KG; ++u) {
      const int j = g + u;
      if (j < nk) {
        const float p = ex2f(fmaf(sc[u], LOG2E, -ms));
        l += p;
#pragma unroll
        for (int c = 0; c < DH; ++c) o[c] = fmaf(p, Vs[j][c], o[c]);
      }
    }
  }
  // merge the 4 warps' partial softmax states (reuse Vs as [warp][lane][DH])
  __syncthreads();
  wm[warp][lane] = m;
  wl[warp][lane] = l;
  float* ob = &Vs[0][0];
  static_assert(AP_WARPS * 32 * DH <= AP_KC * DH * 2, "merge buffer");
  float* mine = (warp < 2 ? &Vs[0][0] : &Ks[0][0]) + ((warp & 1) * 32 + lane) * DH;
  (void)ob;
#pragma unroll
  for (int c = 0; c < DH; ++c) mine[c] = o[c];
  __syncthreads();
  if (warp == 0 && qi < qslot) {
    float mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < AP_WARPS; ++w) mt = fmaxf(mt, wm[w][lane]);
    float lt = 0.f, f[AP_WARPS];
#pragma unroll
    for (int w = 0; w < AP_WARPS; ++w) {
      f[w] = (wm[w][lane] == -INFINITY) ? 0.f : ex2f((wm[w][lane] - mt) * LOG2E);
      lt += wl[w][lane] * f[w];
    }
    const float inv = (live && lt > 0.f) ? 1.0f / lt : 0.f;
    T* orow = out + (size_t)(qb + qi) * out_stride + hoff;
#pragma unroll
    for (int c = 0; c < DH; ++c) {
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < AP_WARPS; ++w) {
        const float* ow = (w < 2 ? &Vs[0][0] : &Ks[0][0]) + ((w & 1) * 32 + lane) * DH;
        a = fmaf(ow[c], f[w], a);
      }
      orow[c] = from_f<T>(a * inv);
    }
  }
}

// ---------------------------------------------------------------------------
// bf16 tensor-core variant of the ragged attention above (DH = 64): same work
// items (sequence, 32-query block), 2 warps x 16 queries; S = Q K^T and
// O += P V on mma.sync m16n8k16 (bf16 in, fp32 accumulate), online softmax
// in the fp32 accumulator fragments, P fed back as the A operand without a
// shared-memory round trip. Keys stream through smem in chunks of 64 (rows
// padded to 72 bf16: conflict-free fragment loads).
// ---------------------------------------------------------------------------
constexpr int AM_WARPS = 2, AM_KC = 64, AM_LD = 72;

__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

__global__ void __launch_bounds__(AM_WARPS * 32) attn_prefill_mma_kernel(
    const int2* __restrict__ items, const bf16* __restrict__ q, int q_stride, const bf16* __restrict__ k,
    const bf16* __restrict__ v, int kv_stride, bf16* __restrict__ out, int out_stride, const int* __restrict__ q_off,
    const int* __restrict__ q_slot, const int* __restrict__ q_len, const int* __restrict__ kv_map,
    const int* __restrict__ kv_off, const int* __restrict__ kv_len, const unsigned char* __restrict__ key_ok,
    int causal, float scale) {
  pdl_enter();
  constexpr int DH = 64;
  __shared__ __align__(16) bf16 Qs[32][AM_LD];
  __shared__ __align__(16) bf16 Ks[AM_KC][AM_LD];
  __shared__ __align__(16) bf16 Vt[DH][AM_LD];
  __shared__ float kbias[AM_KC];
  const int2 it = items[blockIdx.x];
  const int s = it.x, qbeg = it.y * 32, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qslot = q_slot[s];
  const int qlen = q_len[s];
  const int kvs = kv_map ? kv_map[s] : s;
  const int kb = kv_off[kvs];
  const int L = kv_len[kvs];
  const int hoff = h * DH;
  const int qb = q_off[s];
  // Q block -> smem (rows past q_len are zero)
  for (int idx = threadIdx.x; idx < 32 * 8; idx += blockDim.x) {
    const int r = idx >> 3, c8 = (idx & 7) * 8;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (qbeg + r < qlen) u = *reinterpret_cast<const uint4*>(q + (size_t)(qb + qbeg + r) * q_stride + hoff + c8);
    *reinterpret_cast<uint4*>(&Qs[r][c8]) = u;
  }
  __syncthreads();
  // A fragments of this warp's 16 queries, 4 k-steps of 16 dims
  const int g = lane >> 2, tq = lane & 3;
  const int r0 = warp * 16 + g;
  uint32_t qa[4][4];
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int c = ks * 16 + tq * 2;
    qa[ks][0] = *reinterpret_cast<const uint32_t*>(&Qs[r0][c]);
    qa[ks][1] = *reinterpret_cast<const uint32_t*>(&Qs[r0 + 8][c]);
    qa[ks][2] = *reinterpret_cast<const uint32_t*>(&Qs[r0][c + 8]);
    qa[ks][3] = *reinterpret_cast<const uint32_t*>(&Qs[r0 + 8][c + 8]);
  }
  const int qi0 = qbeg + r0, qi1 = qi0 + 8;  // the two query rows this thread accumulates
  float o[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = scale * LOG2E;  // scores kept in log2 units
  const int qmax = min(qslot, qbeg + 32) - 1;
  const int Lc = causal ? min(L, qmax + 1) : L;
  for (int j0 = 0; j0 < Lc; j0 += AM_KC) {
    const int nk = min(AM_KC, Lc - j0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < AM_KC * 8; idx += blockDim.x) {
      const int j = idx >> 3, c8 = (idx & 7) * 8;
      uint4 ku = make_uint4(0, 0, 0, 0), vu = make_uint4(0, 0, 0, 0);
      if (j < nk) {
        const size_t r = (size_t)(kb + j0 + j) * kv_stride + hoff + c8;
        ku = *reinterpret_cast<const uint4*>(k + r);
        vu = *reinterpret_cast<const uint4*>(v + r);
      }
      *reinterpret_cast<uint4*>(&Ks[j][c8]) = ku;
      const bf16* ve = reinterpret_cast<const bf16*>(&vu);
#pragma unroll
      for (int e = 0; e < 8; ++e) Vt[c8 + e][j] = ve[e];
    }
    for (int j = threadIdx.x; j < AM_KC; j += blockDim.x)
      kbias[j] = (j < nk && (key_ok == nullptr || key_ok[kb + j0 + j])) ? 0.f : -INFINITY;
    __syncthreads();
    // S = Q K^T : 16 x 64 per warp (8 n-tiles of 8 keys)
    float sc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t b[2];
        const int kr = n * 8 + g, c = ks * 16 + tq * 2;
        b[0] = *reinterpret_cast<const uint32_t*>(&Ks[kr][c]);
        b[1] = *reinterpret_cast<const uint32_t*>(&Ks[kr][c + 8]);
        mma_bf16_16816(sc[n], qa[ks], b);
      }
    }
    // mask + online softmax (base 2)
    float cm0 = -INFINITY, cm1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = n * 8 + tq * 2 + e;
        const float kbj = kbias[j];
        float a0 = sc[n][e] * sl2 + kbj, a1 = sc[n][2 + e] * sl2 + kbj;
        if (causal && j0 + j > qi0) a0 = -INFINITY;
        if (causal && j0 + j > qi1) a1 = -INFINITY;
        sc[n][e] = a0;
        sc[n][2 + e] = a1;
        cm0 = fmaxf(cm0, a0);
        cm1 = fmaxf(cm1, a1);
      }
    }
    cm0 = fmaxf(cm0, __shfl_xor_sync(0xffffffffu, cm0, 1));
    cm0 = fmaxf(cm0, __shfl_xor_sync(0xffffffffu, cm0, 2));
    cm1 = fmaxf(cm1, __shfl_xor_sync(0xffffffffu, cm1, 1));
    cm1 = fmaxf(cm1, __shfl_xor_sync(0xffffffffu, cm1, 2));
    const float mn0 = fmaxf(m0, cm0), mn1 = fmaxf(m1, cm1);
    const float b0 = mn0 == -INFINITY ? 0.f : mn0, b1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = ex2f(m0 - b0), c1 = ex2f(m1 - b1);
    m0 = mn0;
    m1 = mn1;
    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      sc[n][0] = ex2f(sc[n][0] - b0);
      sc[n][1] = ex2f(sc[n][1] - b0);
      sc[n][2] = ex2f(sc[n][2] - b1);
      sc[n][3] = ex2f(sc[n][3] - b1);
      ps0 += sc[n][0] + sc[n][1];
      ps1 += sc[n][2] + sc[n][3];
    }
    l0 = l0 * c0 + ps0;
    l1 = l1 * c1 + ps1;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      o[n][0] *= c0;
      o[n][1] *= c0;
      o[n][2] *= c1;
      o[n][3] *= c1;
    }
    // O += P V : P fragments straight from the score accumulators
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t pa[4];
      pa[0] = pack_bf16(sc[2 * ks][0], sc[2 * ks][1]);
      pa[1] = pack_bf16(sc[2 * ks][2], sc[2 * ks][3]);
      pa[2] = pack_bf16(sc[2 * ks + 1][0], sc[2 * ks + 1][1]);
      pa[3] = pack_bf16(sc[2 * ks + 1][2], sc[2 * ks + 1][3]);
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        uint32_t b[2];
        const int dr = n * 8 + g, c = ks * 16 + tq * 2;
        b[0] = *reinterpret_cast<const uint32_t*>(&Vt[dr][c]);
        b[1] = *reinterpret_cast<const uint32_t*>(&Vt[dr][c + 8]);
        mma_bf16_16816(o[n], pa, b);
      }
    }
  }
  // row sums across the quad, normalise, store (pad rows of the slot get 0)
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = (qi0 < qlen && l0 > 0.f) ? 1.f / l0 : 0.f;
  const float i1 = (qi1 < qlen && l1 > 0.f) ? 1.f / l1 : 0.f;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    const int c = hoff + n * 8 + tq * 2;
    if (qi0 < qslot)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(qb + qi0) * out_stride + c) =
          __floats2bfloat162_rn(o[n][0] * i0, o[n][1] * i0);
    if (qi1 < qslot)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(qb + qi1) * out_stride + c) =
          __floats2bfloat162_rn(o[n][2] * i1, o[n][3] * i1);
  }
}

// ---------------------------------------------------------------------------
// All-heads variant of the bf16 prefill attention (d_head = 64, heads <= 8):
// one CTA per (sequence, 32-query block) covers every head, so K/V rows are
// fetched once as whole d-wide rows with cp.async (1 KB contiguous per key at
// d = 512) instead of once per head. Warp 2h + i owns head h, queries
// 16i..16i+15; QK^T and PV on mma.sync m16n8k16, V fragments by
// ldmatrix.trans (no scalar transpose), online softmax over 32-key chunks.
// Same item list, masks and output contract as attn_prefill_mma_kernel.
// ---------------------------------------------------------------------------
constexpr int AH_KC = 32, AH_PAD = 8;

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

inline size_t attn_heads_smem(int d) { return (size_t)(32 + 2 * AH_KC) * (d + AH_PAD) * 2 + AH_KC * sizeof(float); }

template <int HT>  // heads per CTA (compile-time: index math by shifts); blockIdx.y = head group
__global__ void __launch_bounds__(512, 2) attn_prefill_heads_kernel(
    const int2* __restrict__ items, const bf16* __restrict__ q, int q_stride, const bf16* __restrict__ k,
    const bf16* __restrict__ v, int kv_stride, bf16* __restrict__ out, int out_stride, const int* __restrict__ q_off,
    const int* __restrict__ q_slot, const int* __restrict__ q_len, const int* __restrict__ kv_map,
    const int* __restrict__ kv_off, const int* __restrict__ kv_len, const unsigned char* __restrict__ key_ok,
    int causal, float scale, int H) {
  pdl_enter();
  constexpr int DH = 64;
  extern __shared__ __align__(16) unsigned char ah_raw[];
  (void)H;
  constexpr int d = HT * DH, ld = d + AH_PAD, c8n = d / 8;
  bf16* Qs = reinterpret_cast<bf16*>(ah_raw);
  bf16* Ks = Qs + 32 * ld;
  bf16* Vs = Ks + AH_KC * ld;
  float* kbias = reinterpret_cast<float*>(Vs + AH_KC * ld);
  const int2 it = items[blockIdx.x];
  const int s = it.x, qbeg = it.y * 32;
  const int tid = threadIdx.x, nthr = blockDim.x;
  {  // head group blockIdx.y: its d columns of q / k / v / out
    const int hg = blockIdx.y * d;
    q += hg;
    k += hg;
    v += hg;
    out += hg;
  }
  const int warp = tid >> 5, lane = tid & 31;
  const int qslot = q_slot[s], qlen = q_len[s];
  const int kvs = kv_map ? kv_map[s] : s;
  const int kb = kv_off[kvs], L = kv_len[kvs], qb = q_off[s];
  // Q block (rows past q_len zero-filled)
  for (int idx = tid; idx < 32 * c8n; idx += nthr) {
    const int r = idx / c8n, c = (idx - r * c8n) * 8;
    const bool ok = qbeg + r < qlen;
    cp_async16_zfill(Qs + r * ld + c, q + (size_t)(qb + (ok ? qbeg + r : 0)) * q_stride + c, ok);
  }
  const int h = warp >> 1, qh = warp & 1, hoff = h * DH;
  const int g = lane >> 2, tq = lane & 3;
  const int qi0 = qbeg + qh * 16 + g, qi1 = qi0 + 8;
  float o[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = scale * LOG2E;
  const int qmax = min(qslot, qbeg + 32) - 1;
  const int Lc = causal ? min(L, qmax + 1) : L;
  uint32_t qa[4][4];
  for (int j0 = 0; j0 < Lc; j0 += AH_KC) {
    const int nk = min(AH_KC, Lc - j0);
    if (j0 > 0) __syncthreads();  // previous chunk consumed
    for (int idx = tid; idx < AH_KC * c8n; idx += nthr) {
      const int j = idx / c8n, c = (idx - j * c8n) * 8;
      const bool ok = j < nk;
      const size_t r = (size_t)(kb + j0 + (ok ? j : 0)) * kv_stride + c;
      cp_async16_zfill(Ks + j * ld + c, k + r, ok);
      cp_async16_zfill(Vs + j * ld + c, v + r, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int j = tid; j < AH_KC; j += nthr)
      kbias[j] = (j < nk && (key_ok == nullptr || key_ok[kb + j0 + j])) ? 0.f : -INFINITY;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    {  // Q fragments re-read from shared memory each chunk (keeps registers for two CTAs per SM)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int c = hoff + ks * 16 + tq * 2;
        const bf16* q0 = Qs + (qh * 16 + g) * ld + c;
        const bf16* q1 = q0 + 8 * ld;
        qa[ks][0] = *reinterpret_cast<const uint32_t*>(q0);
        qa[ks][1] = *reinterpret_cast<const uint32_t*>(q1);
        qa[ks][2] = *reinterpret_cast<const uint32_t*>(q0 + 8);
        qa[ks][3] = *reinterpret_cast<const uint32_t*>(q1 + 8);
      }
    }
    // S = Q K^T: 16 queries x 32 keys (4 n-tiles of 8 keys)
    float sc[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
      const bf16* kr = Ks + (n * 8 + g) * ld + hoff + tq * 2;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t b[2];
        b[0] = *reinterpret_cast<const uint32_t*>(kr + ks * 16);
        b[1] = *reinterpret_cast<const uint32_t*>(kr + ks * 16 + 8);
        mma_bf16_16816(sc[n], qa[ks], b);
      }
    }
    // mask + online softmax (base 2)
    float cm0 = -INFINITY, cm1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < 4; ++n) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = n * 8 + tq * 2 + e;
        const float kbj = kbias[j];
        float a0 = sc[n][e] * sl2 + kbj, a1 = sc[n][2 + e] * sl2 + kbj;
        if (causal && j0 + j > qi0) a0 = -INFINITY;
        if (causal && j0 + j > qi1) a1 = -INFINITY;
        sc[n][e] = a0;
        sc[n][2 + e] = a1;
        cm0 = fmaxf(cm0, a0);
        cm1 = fmaxf(cm1, a1);
      }
    }
    cm0 = fmaxf(cm0, __shfl_xor_sync(0xffffffffu, cm0, 1));
    cm0 = fmaxf(cm0, __shfl_xor_sync(0xffffffffu, cm0, 2));
    cm1 = fmaxf(cm1, __shfl_xor_sync(0xffffffffu, cm1, 1));
    cm1 = fmaxf(cm1, __shfl_xor_sync(0xffffffffu, cm1, 2));
    const float mn0 = fmaxf(m0, cm0), mn1 = fmaxf(m1, cm1);
    const float b0 = mn0 == -INFINITY ? 0.f : mn0, b1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = ex2f(m0 - b0), c1 = ex2f(m1 - b1);
    m0 = mn0;
    m1 = mn1;
    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      sc[n][0] = ex2f(sc[n][0] - b0);
      sc[n][1] = ex2f(sc[n][1] - b0);
      sc[n][2] = ex2f(sc[n][2] - b1);
      sc[n][3] = ex2f(sc[n][3] - b1);
      ps0 += sc[n][0] + sc[n][1];
      ps1 += sc[n][2] + sc[n][3];
    }
    l0 = l0 * c0 + ps0;
    l1 = l1 * c1 + ps1;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      o[n][0] *= c0;
      o[n][1] *= c0;
      o[n][2] *= c1;
      o[n][3] *= c1;
    }
    // O += P V: P fragments from the score accumulators, V fragments by ldmatrix.trans
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t pa[4];
      pa[0] = pack_bf16(sc[2 * ks][0], sc[2 * ks][1]);
      pa[1] = pack_bf16(sc[2 * ks][2], sc[2 * ks][3]);
      pa[2] = pack_bf16(sc[2 * ks + 1][0], sc[2 * ks + 1][1]);
      pa[3] = pack_bf16(sc[2 * ks + 1][2], sc[2 * ks + 1][3]);
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        // lanes 0-15: keys ks*16 + lane, dims n*8..; lanes 16-31: same keys, dims (n+1)*8..
        const bf16* vp = Vs + (ks * 16 + (lane & 15)) * ld + hoff + (n + (lane >> 4)) * 8;
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(vp));
        uint32_t b[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "r"(sa));
        mma_bf16_16816(o[n], pa, b);
        mma_bf16_16816(o[n + 1], pa, b + 2);
      }
    }
  }
  if (Lc <= 0) __syncthreads();  // (no chunk ran: keep the Q copy's barrier discipline)
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = (qi0 < qlen && l0 > 0.f) ? 1.f / l0 : 0.f;
  const float i1 = (qi1 < qlen && l1 > 0.f) ? 1.f / l1 : 0.f;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    const int c = hoff + n * 8 + tq * 2;
    if (qi0 < qslot)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(qb + qi0) * out_stride + c) =
          __floats2bfloat162_rn(o[n][0] * i0, o[n][1] * i0);
    if (qi1 < qslot)
      *reinterpret_cast<__nv_bfloat162*>(out + (size_t)(qb + qi1) * out_stride + c) =
          __floats2bfloat162_rn(o[n][2] * i1, o[n][3] * i1);
  }
}

// ---------------------------------------------------------------------------
// Decode attention, one CTA per Stage-I row covering every head (bf16,
// d_head = 64, heads <= 16): the row's key/value rows (all heads, d wide and
// contiguous) are staged through shared memory in 32-key chunks with
// cp.async, so each key row is one coalesced d*2-byte transfer instead of
// per-head strided reads; warp h then runs head h with one key per lane for
// QK^T and two head dims per lane for PV (online softmax across chunks).
// SELF: appends this step's k/v at cache slot t (history slot j of logical row
// r lives in physical row hist[r * cap + j], or row r when hist == nullptr).
// CROSS: attends the row's sentence memory keys (computed once in encode).
// Same arguments and results as attn_decode_kernel (infer.py:259-285).
// ---------------------------------------------------------------------------
constexpr int AD_KC = 32, AD_PAD = 8;

inline size_t attn_rows_smem(int d) {
  return (size_t)2 * AD_KC * (d + AD_PAD) * 2 + (size_t)d * sizeof(float) + AD_KC * sizeof(int);
}

template <bool SELF, int HT>  // HT: heads (compile-time index math)
__global__ void __launch_bounds__(512) attn_decode_rows_kernel(
    const bf16* __restrict__ q, int q_stride, const bf16* __restrict__ knew, const bf16* __restrict__ vnew,
    int new_stride, bf16* __restrict__ kc, bf16* __restrict__ vc, int c_stride, const int* __restrict__ hist_a,
    const int* __restrict__ hist_b, int cap, int t, const int* __restrict__ t_dev, const int* __restrict__ row_seq,
    const int* __restrict__ kv_off, const int* __restrict__ kv_len, const int* __restrict__ R_dev, int R, int heads,
    float scale, bf16* __restrict__ out, int out_stride, int kv_prefetch) {
  pdl_trigger();
  constexpr int DH = 64;
  extern __shared__ __align__(16) unsigned char ad_raw[];
  constexpr int d = HT * DH, ld = d + AD_PAD, c8n = d / 8;
  constexpr int heads_c = HT;
  bf16* Ks = reinterpret_cast<bf16*>(ad_raw);
  bf16* Vs = Ks + AD_KC * ld;
  float* qs = reinterpret_cast<float*>(Vs + AD_KC * ld);
  int* hs = reinterpret_cast<int*>(qs + d);
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31;
  uint64_t kv_pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kv_pol));
  const int r = blockIdx.x;
  // cross attention with kv_prefetch: the sentence memory (immutable during
  // Stage I) streams its first key chunk into shared memory before the
  // grid-dependency wait, overlapping the previous kernel
  bool pre = false;
  if (!SELF && kv_prefetch && r < R) {
    const int sq = row_seq ? row_seq[r] : r;
    const int nk0 = min(AD_KC, kv_len[sq]);
    const size_t row0 = kv_off[sq];
    for (int idx = tid; idx < nk0 * c8n; idx += nthr) {
      const int j = idx / c8n, c = (idx - j * c8n) * 8;
      const size_t pr = (row0 + j) * (size_t)new_stride + c;
      const uint32_t sk = static_cast<uint32_t>(__cvta_generic_to_shared(Ks + j * ld + c));
      const uint32_t sv = static_cast<uint32_t>(__cvta_generic_to_shared(Vs + j * ld + c));
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sk), "l"(knew + pr),
                   "l"(kv_pol)
                   : "memory");
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sv), "l"(vnew + pr),
                   "l"(kv_pol)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    pre = true;
  }
  pdl_wait();
  // the query row is requested before the device row count / step resolve (the
  // grid never exceeds the launch's host bound, which the buffer holds)
  constexpr int QPT = (d + 63) / 64;  // >= d / blockDim.x for blockDim.x >= 64
  float qv[QPT];
#pragma unroll
  for (int i = 0; i < QPT; ++i) {
    const int c = tid + i * nthr;
    qv[i] = c < d ? to_f(q[(size_t)r * q_stride + c]) * scale : 0.f;
  }
  if (R_dev) R = *R_dev;
  if (t_dev) t = *t_dev;
  if (r >= R) {
    asm volatile("cp.async.wait_all;" ::: "memory");  // no copy may outlive the CTA
    return;
  }
  (void)heads;
  const int* __restrict__ hist = (hist_b != nullptr && (t & 1)) ? hist_b : hist_a;
  int L;
  size_t kv_row0 = 0;
  if (SELF) {
    L = t + 1;
    // append this step's k / v at slot t (all heads)
    const size_t dst = ((size_t)r * cap + t) * c_stride;
    for (int c = tid; c < c8n; c += nthr) {
      *reinterpret_cast<uint4*>(kc + dst + c * 8) = *reinterpret_cast<const uint4*>(knew + (size_t)r * new_stride + c * 8);
      *reinterpret_cast<uint4*>(vc + dst + c * 8) = *reinterpret_cast<const uint4*>(vnew + (size_t)r * new_stride + c * 8);
    }
  } else {
    const int sq = row_seq ? row_seq[r] : r;
    L = kv_len[sq];
    kv_row0 = kv_off[sq];
  }
#pragma unroll
  for (int i = 0; i < QPT; ++i) {
    const int c = tid + i * nthr;
    if (c < d) qs[c] = qv[i];
  }
  const int h = warp;
  const bool active = h < heads_c;
  float m = -INFINITY, l = 0.f, o0 = 0.f, o1 = 0.f;
  for (int j0 = 0; j0 < L; j0 += AD_KC) {
    const int nk = min(AD_KC, L - j0);
    __syncthreads();  // previous chunk consumed (and qs / the cache append visible)
    if (SELF && hist) {
      for (int j = tid; j < nk; j += nthr) hs[j] = hist[(size_t)r * cap + j0 + j];
      __syncthreads();
    }
    for (int idx = tid; idx < ((pre && j0 == 0) ? 0 : nk * c8n); idx += nthr) {  // chunk 0 prefetched
      const int j = idx / c8n, c = (idx - j * c8n) * 8;
      const bf16* ksrc;
      const bf16* vsrc;
      if (SELF) {
        const int jj = j0 + j;
        if (jj == t) {
          ksrc = knew + (size_t)r * new_stride + c;
          vsrc = vnew + (size_t)r * new_stride + c;
        } else {
          const size_t pr = ((size_t)(hist ? hs[j] : r) * cap + jj) * c_stride + c;
          ksrc = kc + pr;
          vsrc = vc + pr;
        }
      } else {
        const size_t pr = (kv_row0 + j0 + j) * (size_t)new_stride + c;
        ksrc = knew + pr;
        vsrc = vnew + pr;
      }
      const uint32_t sk = static_cast<uint32_t>(__cvta_generic_to_shared(Ks + j * ld + c));
      const uint32_t sv = static_cast<uint32_t>(__cvta_generic_to_shared(Vs + j * ld + c));
      // K/V streams (every row's history / sentence memory, read once per step)
      // are marked evict-first so they do not push the L2-resident decoder and
      // vocabulary weights (evict-last) out of L2
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sk), "l"(ksrc), "l"(kv_pol)
                   : "memory");
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sv), "l"(vsrc), "l"(kv_pol)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (active) {
      // scores: lane = key of the chunk (same dot order as attn_decode_kernel)
      float s = -INFINITY;
      if (lane < nk) {
        const bf16* kr = Ks + lane * ld + h * DH;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < DH; c += 8) {
          float kk[8];
          load8(kr + c, kk);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            a0 = fmaf(qs[h * DH + c + e], kk[e], a0);
            a1 = fmaf(qs[h * DH + c + e + 1], kk[e + 1], a1);
          }
        }
        s = a0 + a1;
      }
      const float mn = fmaxf(m, warp_max(s));
      const float sc = ex2f((m - mn) * LOG2E);  // first chunk: m = -inf -> 0
      const float p = lane < nk ? ex2f((s - mn) * LOG2E) : 0.f;
      l = l * sc + warp_sum(p);
      m = mn;
      o0 *= sc;
      o1 *= sc;
      const bf16* vcol = Vs + h * DH + 2 * lane;
      for (int i = 0; i < nk; ++i) {
        const float pi = __shfl_sync(0xffffffffu, p, i);
        const float2 v2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vcol + i * ld));
        o0 = fmaf(pi, v2.x, o0);
        o1 = fmaf(pi, v2.y, o1);
      }
    }
  }
  if (active) {
    const float inv = 1.0f / l;
    *reinterpret_cast<__nv_bfloat162*>(out + (size_t)r * out_stride + h * DH + 2 * lane) =
        __floats2bfloat162_rn(o0 * inv, o1 * inv);
  }
}

// ---------------------------------------------------------------------------
// Single-query attention for one Stage-I decoder step (infer.py:259-285).
// SELF: append this step's k/v at cache slot t, then attend slots 0..t of the
//       row's history; history slot j of logical row r lives in physical row
//       hist[r * cap + j] (beam reorder = index permutation, infer.py:307-318).
// CROSS: attend the row's sentence memory keys (computed once in encode).
// One warp per (row, head); q in registers; lanes own keys for QK (16 B
// vector loads) and head dims for PV (coalesced rows).
// ---------------------------------------------------------------------------
template <typename T, int DH, bool SELF>
__global__ void __launch_bounds__(128) attn_decode_kernel(
    const T* __restrict__ q, int q_stride, const T* __restrict__ knew, const T* __restrict__ vnew, int new_stride,
    T* __restrict__ kc, T* __restrict__ vc, int c_stride, const int* __restrict__ hist_a,
    const int* __restrict__ hist_b, int cap, int t, const int* __restrict__ t_dev, const int* __restrict__ row_seq,
    const int* __restrict__ kv_off,
    const int* __restrict__ kv_len, const int* __restrict__ R_dev, int R, int heads, int lk_max, float scale,
    T* __restrict__ out, int out_stride, int kv_prefetch) {
  pdl_trigger();
  extern __shared__ float sm[];
  // Cross attention with kv_prefetch: the sentence memory K/V (and the row ->
  // sentence metadata) are never written during Stage I, so the first 32 keys'
  // K fragments are requested before the grid-dependency wait and overlap the
  // previous kernel (the caller guarantees the encoder finished before Stage I).
  constexpr bool PRE = !SELF && std::is_same<T, bf16>::value && DH % 8 == 0;
  uint4 kpre[PRE ? DH / 8 : 1];
  bool have_pre = false;
  if constexpr (PRE) {
    const int item0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int r0 = item0 / heads, h0 = item0 - r0 * heads;
    if (kv_prefetch && r0 < R) {
      const int sq = row_seq ? row_seq[r0] : r0;
      const int L0 = kv_len[sq];
      const int ln = threadIdx.x & 31;
      if (ln < L0) {
        const T* kr = knew + ((size_t)kv_off[sq] + ln) * new_stride + h0 * DH;
#pragma unroll
        for (int c = 0; c < DH / 8; ++c) kpre[c] = *reinterpret_cast<const uint4*>(kr + 8 * c);
      }
      have_pre = true;
    }
  }
  pdl_wait();
  constexpr int DPL = DH >= 32 ? DH / 32 : 1;
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * nwarp + warp;
  // the query row is requested before the device row count / step resolve
  // (row clamped to the launch's host bound; items past the live rows exit below)
  const int r = min(item / heads, R - 1), h = item - (item / heads) * heads;
  const int hoff = h * DH;
  float qr[DH];
  {
    const T* src = q + (size_t)r * q_stride + hoff;
    if (DH % 8 == 0) {
#pragma unroll
      for (int c = 0; c < DH; c += 8) load8(src + c, qr + c);
    } else {
#pragma unroll
      for (int c = 0; c < DH; ++c) qr[c] = to_f(src[c]);
    }
#pragma unroll
    for (int c = 0; c < DH; ++c) qr[c] *= scale;
  }
  if (R_dev) R = *R_dev;
  if (t_dev) t = *t_dev;
  if (item >= R * heads) return;
  // beam decoding ping-pongs the history map by step parity (reorder writes the other one)
  const int* __restrict__ hist = (hist_b != nullptr && (t & 1)) ? hist_b : hist_a;  // nullptr: identity
  float* sc = sm + warp * lk_max;
  int L;
  size_t kv_row0 = 0;
  if (SELF) {
    L = t + 1;
    const size_t dst = ((size_t)r * cap + t) * c_stride + hoff;
    for (int c = lane; c < DH; c += 32) {
      kc[dst + c] = knew[(size_t)r * new_stride + hoff + c];
      vc[dst + c] = vnew[(size_t)r * new_stride + hoff + c];
    }
  } else {
    const int sq = row_seq ? row_seq[r] : r;
    L = kv_len[sq];
    kv_row0 = kv_off[sq];
  }
  // history row of slot j (hist == nullptr: identity, greedy rows never reorder)
  auto hrow = [&](int j) -> size_t { return hist ? (size_t)hist[(size_t)r * cap + j] : (size_t)r; };
  auto krow = [&](int j) -> const T* {
    if (SELF)
      return (j == t) ? knew + (size_t)r * new_stride + hoff : kc + (hrow(j) * cap + j) * c_stride + hoff;
    return knew + (kv_row0 + j) * (size_t)new_stride + hoff;
  };
  auto vrow = [&](int j) -> const T* {
    if (SELF)
      return (j == t) ? vnew + (size_t)r * new_stride + hoff : vc + (hrow(j) * cap + j) * c_stride + hoff;
    return vnew + (kv_row0 + j) * (size_t)new_stride + hoff;
  };
  // PV mapping (see below); the first VPRE keys' V fragments are requested now,
  // before the scores, so their latency overlaps QK^T and the softmax
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int LPG = DH / VEC >= 1 ? DH / VEC : 1;
  constexpr int G = 32 / LPG;
  constexpr int VPRE = 8;
  const int grp = lane / LPG, li = lane % LPG;
  uint4 vpre[VPRE];
  if (DH % VEC == 0 && LPG * VEC == DH) {
#pragma unroll
    for (int m = 0; m < VPRE; ++m) {
      const int j = min(grp + G * m, L - 1);
      vpre[m] = *reinterpret_cast<const uint4*>(vrow(j) + li * VEC);
    }
  }
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) {
    const T* kr = krow(j);
    float a0 = 0.f, a1 = 0.f;
    if (DH % 8 == 0) {
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        float kk[8];
        if constexpr (PRE) {
          if (have_pre && j == lane) {  // prefetched fragment (same conversion as load8)
            const __nv_bfloat162* hp = reinterpret_cast<const __nv_bfloat162*>(&kpre[c / 8]);
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
              const float2 f = __bfloat1622float2(hp[i2]);
              kk[2 * i2] = f.x;
              kk[2 * i2 + 1] = f.y;
            }
          } else {
            load8(kr + c, kk);
          }
        } else {
          load8(kr + c, kk);
        }
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          a0 = fmaf(qr[c + e], kk[e], a0);
          a1 = fmaf(qr[c + e + 1], kk[e + 1], a1);
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < DH; ++c) a0 = fmaf(qr[c], to_f(kr[c]), a0);
    }
    const float a = a0 + a1;
    sc[j] = a;
    mx = fmaxf(mx, a);
  }
  mx = warp_max(mx);
  float sum = 0.f;
  const float ms = mx * LOG2E;
  for (int j = lane; j < L; j += 32) {
    const float e = ex2f(fmaf(sc[j], LOG2E, -ms));
    sc[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.0f / sum;
  // PV: G groups of LPG lanes; group g takes keys j = g, g+G, ...; a lane owns
  // VEC consecutive head dims and loads them as one 16-byte vector per key.
  float acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
  int j_start = grp;
  if (DH % VEC == 0 && LPG * VEC == DH) {
#pragma unroll
    for (int m = 0; m < VPRE; ++m) {
      const int j = grp + G * m;
      if (j < L) {
        const float p = sc[j];
        float vv[VEC];
        const T* pv = reinterpret_cast<const T*>(&vpre[m]);
#pragma unroll
        for (int e = 0; e < VEC; ++e) vv[e] = to_f(pv[e]);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fmaf(p, vv[e], acc[e]);
      }
    }
    j_start = grp + G * VPRE;
  }
#pragma unroll 4
  for (int j = j_start; j < L; j += G) {
    const float p = sc[j];
    float vv[VEC];
    loadvec(vrow(j) + li * VEC, vv);
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = fmaf(p, vv[e], acc[e]);
  }
#pragma unroll
  for (int o = LPG; o < 32; o <<= 1)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (grp == 0) {
    T* dst = out + (size_t)r * out_stride + hoff + li * VEC;
#pragma unroll
    for (int e = 0; e < VEC; ++e) dst[e] = from_f<T>(acc[e] * inv);
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


// Per-thread running accumulator over a contiguous run of columns of one row:
// running max / rescaled sum of exp (online softmax) and a top-KT list
// ordered (value desc, id asc).
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
  // bubble (v, c) into the sorted list with static indices only, so the
  // list stays in registers (a dynamic insert position spills it to local memory)
  __device__ __forceinline__ void insert(float v, int c) {
    if (!better(v, c, val[KT - 1], id[KT - 1])) return;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      const bool b = better(v, c, val[i], id[i]);
      const float tv = b ? val[i] : v;
      const int tc = b ? id[i] : c;
      val[i] = b ? v : val[i];
      id[i] = b ? c : id[i];
      v = tv;
      c = tc;
    }
  }
  // fold a new normaliser max in, rescaling the running sum
  __device__ __forceinline__ void rebase(float cm) {
    if (cm > mx) {
      sum *= ex2f((mx - cm) * LOG2E);
      mx = cm;
    }
  }
  // one column (generic path)
  __device__ __forceinline__ void add1(float x, int c, int norm_allowed) {
    const bool ok = id_allowed(c);
    if (ok) insert(x, c);
    if (norm_allowed && !ok) return;
    rebase(x);
    sum += ex2f((x - mx) * LOG2E);
  }
  // 32 columns col0..col0+31, all generable (col0 >= 32): tree reductions
  // so the per-element work is independent (ILP) -- the epilogue thread
  // owns a whole row, so dependency chains would otherwise dominate.
  __device__ __forceinline__ void add32_fast(const float* v, int col0) {
    float mv[16];
    int mi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool b = v[i + 16] > v[i];
      mv[i] = b ? v[i + 16] : v[i];
      mi[i] = b ? i + 16 : i;
    }
#pragma unroll
    for (int st = 8; st > 0; st >>= 1) {
#pragma unroll
      for (int i = 0; i < st; ++i) {
        const bool b = better(mv[i + st], mi[i + st], mv[i], mi[i]);
        mv[i] = b ? mv[i + st] : mv[i];
        mi[i] = b ? mi[i + st] : mi[i];
      }
    }
    const float cm = mv[0];
    if (KT == 1) {
      if (better(cm, col0 + mi[0], val[0], id[0])) {
        val[0] = cm;
        id[0] = col0 + mi[0];
      }
    } else if (better(cm, col0 + mi[0], val[KT - 1], id[KT - 1])) {
#pragma unroll
      for (int i = 0; i < 32; ++i) insert(v[i], col0 + i);
    }
    rebase(cm);
    const float ms = mx * LOG2E;
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 32; ++i) s4[i & 3] += ex2f(fmaf(v[i], LOG2E, -ms));
    sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
};

// tcgen05 epilogue: one thread owns one row of a 128 x BN logits tile.
template <int KT>
struct VocabEpi {
  static constexpr bool kRowWise = true;
  VocabParts parts;
  int norm_allowed;
  int bn;
  struct State {
    TileAcc<KT> acc;
  };
  __device__ __forceinline__ void begin(State& s, int, int) const { s.acc.init(); }
  __device__ __forceinline__ void chunk(State& s, int row, int col0, const float* v, int n) const {
    if (col0 >= 32 && n == 32) {
      s.acc.add32_fast(v, col0);
      return;
    }
    if (col0 == 0) parts.eos[row] = v[EOS_ID];
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < n) s.acc.add1(v[i], col0 + i, norm_allowed);
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
  pdl_enter();
  const int row = blockIdx.x, tile = blockIdx.y, lane = threadIdx.x;
  const int src = row_map ? row_map[row] : row;
  const float* l = logits + (size_t)src * ld;
  const int c0 = tile * tile_w, c1 = min(V, c0 + tile_w);
  TileAcc<KT> a;
  a.init();
  for (int c = c0 + lane; c < c1; c += 32) {
    const float x = l[c];
    a.add1(x, c, norm_allowed);
    if (c == EOS_ID) parts.eos[row] = x;
  }
  // merge lanes: max + rescaled sum
  const float m = warp_max(a.mx);
  float s = (a.mx == -INFINITY) ? 0.f : a.sum * ex2f((a.mx - m) * LOG2E);
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

// Top-1 merge (greedy selection / Stage-II argmax): every partial field of a
// lane's tiles is loaded in one pass (one dependent round trip), then the
// lane's online {max, sum} and best (value desc, id asc) are warp-reduced.
// Same results as merge_row<KT>(parts, row, 1): identical max and order of
// the rescaled sums per lane, identical tie rule.
template <bool CG = false>
__device__ __forceinline__ RowStat merge_row1(const VocabParts& parts, int row) {
  const int lane = threadIdx.x & 31;
  // CG: the partials were written by other CTAs of the running grid (fused selection tail)
  auto ldp = [](const auto* q) { return CG ? __ldcg(q) : *q; };
  const size_t base = (size_t)row * parts.ntiles;
  constexpr int MAXP = 8;  // tiles per lane held in registers (ntiles <= 256)
  float pm[MAXP], ps[MAXP], pv[MAXP];
  int pi[MAXP];
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    const int t = lane + 32 * i;
    const bool ok = t < parts.ntiles;
    const size_t o = base + (ok ? t : 0);
    pm[i] = ok ? ldp(parts.mx + o) : -INFINITY;
    ps[i] = ok ? ldp(parts.sum + o) : 0.f;
    pv[i] = ok ? ldp(parts.val + o) : -INFINITY;
    pi[i] = ok ? ldp(parts.id + o) : 0x7fffffff;
  }
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXP; ++i) m = fmaxf(m, pm[i]);
  for (int t = lane + 32 * MAXP; t < parts.ntiles; t += 32) m = fmaxf(m, ldp(parts.mx + base + t));
  m = warp_max(m);
  float sm = 0.f, bv = -INFINITY;
  int bi = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    if (pm[i] != -INFINITY) sm += ps[i] * ex2f((pm[i] - m) * LOG2E);
    if (pi[i] != 0x7fffffff && better(pv[i], pi[i], bv, bi)) {
      bv = pv[i];
      bi = pi[i];
    }
  }
  for (int t = lane + 32 * MAXP; t < parts.ntiles; t += 32) {
    const float tm = ldp(parts.mx + base + t);
    if (tm != -INFINITY) sm += ldp(parts.sum + base + t) * ex2f((tm - m) * LOG2E);
    const float v = ldp(parts.val + base + t);
    const int id = ldp(parts.id + base + t);
    if (id != 0x7fffffff && better(v, id, bv, bi)) {
      bv = v;
      bi = id;
    }
  }
  sm = warp_sum(sm);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  RowStat rs;
  rs.mx = m;
  rs.lse = logf(sm);
  rs.eos = parts.eos[row];
  rs.kt = 1;
  rs.val[0] = bv;
  rs.id[0] = bi;
  return rs;
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
    if (tm != -INFINITY) s += parts.sum[base + t] * ex2f((tm - m) * LOG2E);
  }
  s = warp_sum(s);
  RowStat rs;
  rs.mx = m;
  rs.lse = logf(s);
  rs.eos = parts.eos[row];
  rs.kt = kt;
  // kt <= KT rounds of a k-way merge: every lane holds a cursor into each of its
  // (<= 8) tiles' sorted top-KT lists and that tile's current head in registers; a
  // round takes the warp-best head (lowest id on ties), and only the owning lane
  // advances that tile's cursor (one load) -- no list is rescanned.
  constexpr int MAXP = 8;
  if (parts.ntiles > 32 * MAXP) {  // (not reached for V <= 32768: at most 256 tiles per row)
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
            break;
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
  float hv[MAXP];
  int hid[MAXP], cur[MAXP];
#pragma unroll
  for (int i = 0; i < MAXP; ++i) {
    const int t = lane + 32 * i;
    cur[i] = 0;
    hv[i] = -INFINITY;
    hid[i] = 0x7fffffff;
    if (t < parts.ntiles) {
      hv[i] = parts.val[(base + t) * KT];
      hid[i] = parts.id[(base + t) * KT];
    }
  }
  for (int r = 0; r < kt; ++r) {
    float bv = -INFINITY;
    int bid = 0x7fffffff, bslot = -1;
#pragma unroll
    for (int i = 0; i < MAXP; ++i)
      if (hid[i] != 0x7fffffff && better(hv[i], hid[i], bv, bid)) {
        bv = hv[i];
        bid = hid[i];
        bslot = i;
      }
    float wv = bv;
    int wid = bid;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, wv, o);
      const int oid = __shfl_xor_sync(0xffffffffu, wid, o);
      if (better(ov, oid, wv, wid)) {
        wv = ov;
        wid = oid;
      }
    }
    rs.val[r] = wv;
    rs.id[r] = wid;
    if (wid == 0x7fffffff) continue;  // fewer generable candidates than kt (caller handles)
    // the owner of the winning head advances that tile's cursor (ids are unique across tiles)
#pragma unroll
    for (int i = 0; i < MAXP; ++i)
      if (i == bslot && bid == wid) {
        const int t = lane + 32 * i;
        cur[i] += 1;
        if (cur[i] < KT) {
          hv[i] = parts.val[(base + t) * KT + cur[i]];
          hid[i] = parts.id[(base + t) * KT + cur[i]];
        } else {
          hv[i] = -INFINITY;
          hid[i] = 0x7fffffff;
        }
      }
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
// Device-side Stage-I loop control: the step kernels read the current step,
// live-row count and position from here, so one captured step graph serves
// every step (conditional WHILE node; stage1_advance_kernel steps it).
struct StepCtl {
  int t;         // current step
  int R;         // rows alive at step t (prefix of the cap-sorted batch)
  int pos;       // fed position t * k
  int k;
  int max_cap;   // steps to run at most
  int nrows;     // rows in the batch
  int finished;  // rows finished so far
  int pad;       // rows computed so far (plain unrolled graphs)
};

struct GreedyState {
  // next-step embedding (x = E[tok] * sqrt(d) + PE[(t+1) k], y = LN1(x)),
  // fused into the selection so Stage I needs no separate embed kernel
  const void* E;
  const float* pe;
  const float* ln_g;
  const float* ln_b;
  float* x;
  void* y;
  float scale;
  int d;
  int* feed;       // [rows] next fed token
  int* done;       // [rows]
  int* nsteps;     // [rows] steps taken when finished
  int* forced;     // [rows]
  double* score;   // [rows]
  int* anchors;    // [rows][cap]
  const int* caps; // [rows] Stage-I step cap (max_steps)
  int cap;
};

// Embedding + LayerNorm of one row by one warp (generic d <= 1024):
//   x = E[tok] * sqrt(d) + PE[pos] (fp32, unfused mul/add as the reference),
//   y = LN1(x).  d % 256 == 0 takes the vectorised path (8 elements / lane / chunk).
template <typename T, int NC>
__device__ __forceinline__ void warp_embed_ln_vec(const T* __restrict__ E, const float* __restrict__ pe,
                                                  const float* __restrict__ g, const float* __restrict__ b,
                                                  float scale, int d, int tok, int pos, float* __restrict__ x,
                                                  T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  float v[NC][8];
  float4 gq[NC][2], bq[NC][2];  // gain / bias issued with the embedding row (one round trip)
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = (lane + 32 * c) * 8;
    gq[c][0] = __ldg(reinterpret_cast<const float4*>(g + j));
    gq[c][1] = __ldg(reinterpret_cast<const float4*>(g + j + 4));
    bq[c][0] = __ldg(reinterpret_cast<const float4*>(b + j));
    bq[c][1] = __ldg(reinterpret_cast<const float4*>(b + j + 4));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = (lane + 32 * c) * 8;
    float e8[8];
    load8(E + (size_t)tok * d + j, e8);
    const float4 p0 = *reinterpret_cast<const float4*>(pe + (size_t)pos * d + j);
    const float4 p1 = *reinterpret_cast<const float4*>(pe + (size_t)pos * d + j + 4);
    const float pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[c][e] = __fadd_rn(__fmul_rn(e8[e], scale), pp[e]);
      s += v[c][e];
    }
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float a = v[c][e] - mean;
      q += a * a;
    }
  const float inv = 1.0f / sqrtf(warp_sum(q) / d + 1e-5f);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = (lane + 32 * c) * 8;
    const float gg[8] = {gq[c][0].x, gq[c][0].y, gq[c][0].z, gq[c][0].w, gq[c][1].x, gq[c][1].y, gq[c][1].z, gq[c][1].w};
    const float bb[8] = {bq[c][0].x, bq[c][0].y, bq[c][0].z, bq[c][0].w, bq[c][1].x, bq[c][1].y, bq[c][1].z, bq[c][1].w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[c][e] - mean) * inv * gg[e] + bb[e];
    *reinterpret_cast<float4*>(x + j) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
    *reinterpret_cast<float4*>(x + j + 4) = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
    store4v<T>(y + j, make_float4(o[0], o[1], o[2], o[3]));
    store4v<T>(y + j + 4, make_float4(o[4], o[5], o[6], o[7]));
  }
}

template <typename T>
__device__ __forceinline__ void warp_embed_ln(const T* __restrict__ E, const float* __restrict__ pe,
                                              const float* __restrict__ g, const float* __restrict__ b, float scale,
                                              int d, int tok, int pos, float* __restrict__ x, T* __restrict__ y) {
  if (d == 512) return warp_embed_ln_vec<T, 2>(E, pe, g, b, scale, d, tok, pos, x, y);
  if (d == 1024) return warp_embed_ln_vec<T, 4>(E, pe, g, b, scale, d, tok, pos, x, y);
  if (d == 256) return warp_embed_ln_vec<T, 1>(E, pe, g, b, scale, d, tok, pos, x, y);
  const int lane = threadIdx.x & 31;
  float v[32];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int j = lane + 32 * i;
    v[i] = 0.f;
    if (j < d) {
      v[i] = __fadd_rn(__fmul_rn(to_f(E[(size_t)tok * d + j]), scale), pe[(size_t)pos * d + j]);
      s += v[i];
    }
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      const float c = v[i] - mean;
      q += c * c;
    }
  }
  const float inv = 1.0f / sqrtf(warp_sum(q) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int j = lane + 32 * i;
    if (j < d) {
      x[j] = v[i];
      y[j] = from_f<T>((v[i] - mean) * inv * g[j] + b[j]);
    }
  }
}

template <typename T, int NPL>
__global__ void embed_ln_kernel(const int* __restrict__ ids, const int* __restrict__ pos, int pos_const,
                                const int* __restrict__ pos_dev, const int* __restrict__ M_dev, int M, int d,
                                float scale, const T* __restrict__ E, const float* __restrict__ pe,
                                const float* __restrict__ g, const float* __restrict__ b, float* __restrict__ x,
                                T* __restrict__ y) {
  pdl_enter();
  if (M_dev) M = *M_dev;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= M) return;
  const int p = pos ? pos[row] : (pos_dev ? *pos_dev : pos_const);
  warp_embed_ln<T>(E, pe, g, b, scale, d, ids[row], p, x + (size_t)row * d, y + (size_t)row * d);
}

// Selection of one row by one warp (decoding.py:102-150 at beam 1): the
// row's token (warp-uniform), its score / anchor / finish bookkeeping; *fin =
// the row finished at this step.
__device__ __forceinline__ int greedy_pick_row(const RowStat& rs, const GreedyState& st, int row, int t, int done_v,
                                               StepCtl* ctl, int* fin) {
  const int lane = threadIdx.x & 31;
  *fin = 0;
  if (done_v) return st.feed[row];  // finished rows keep feeding EOS (outputs ignored)
  int tok = 0;
  if (lane == 0) {
    const bool last = (t == st.caps[row] - 1);
    int best = rs.id[0];
    float bl = rs.val[0];
    if (best == 0x7fffffff) {  // non-finite logits: finish the row rather than emit a bogus id
      best = EOS_ID;
      bl = rs.eos;
    }
    tok = last ? EOS_ID : best;
    const float logit = last ? rs.eos : bl;
    const float lp = (logit - rs.mx) - rs.lse;
    st.score[row] += (double)lp;
    st.anchors[(size_t)row * st.cap + t] = tok;
    st.feed[row] = tok;
    if (tok == EOS_ID) {
      st.done[row] = 1;
      st.nsteps[row] = t + 1;
      st.forced[row] = last ? 1 : 0;
      if (ctl) atomicAdd(&ctl->finished, 1);
    }
  }
  tok = __shfl_sync(0xffffffffu, tok, 0);
  *fin = tok == EOS_ID;
  return tok;
}

// ... and the next step's embedding x = E[tok] * sqrt(d) + PE[(t + 1) k], y = LN1(x)
template <typename T>
__device__ __forceinline__ void greedy_embed_row(const GreedyState& st, int row, int t, int k, int tok) {
  if (st.x != nullptr)
    warp_embed_ln<T>(static_cast<const T*>(st.E), st.pe, st.ln_g, st.ln_b, st.scale, st.d, tok, (t + 1) * k,
                     st.x + (size_t)row * st.d, static_cast<T*>(st.y) + (size_t)row * st.d);
}

template <typename T, int KT>
__global__ void greedy_select_kernel(VocabParts parts, GreedyState st, int R, int t, int k, StepCtl* ctl) {
  pdl_enter();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // the row's partials, done flag and the step control are requested together
  // (row clamped to the launch's host bound; rows past the live count exit below)
  const int rr = min(row, R - 1);
  StepCtl c{};
  if (ctl) c = *ctl;
  const int done_v = st.done[rr];
  const RowStat rs = KT == 1 ? merge_row1(parts, rr) : merge_row<KT>(parts, rr, 1);
  if (ctl) {
    R = c.R;
    t = c.t;
    k = c.k;
  }
  if (row >= R) return;
  int fin;
  const int tok = greedy_pick_row(rs, st, row, t, done_v, ctl, &fin);
  greedy_embed_row<T>(st, row, t, k, tok);
}

// End of one graph-resident Stage-I step: advance the control block and
// decide whether the WHILE node runs another step (decoding.py:102, :149).
__global__ void stage1_advance_kernel(StepCtl* ctl, const int* __restrict__ alive,
                                      cudaGraphConditionalHandle handle) {
  pdl_enter();
  const int t = ctl->t + 1;
  const bool more = t < ctl->max_cap && ctl->finished < ctl->nrows && alive[t] > 0;
  if (more) {
    ctl->t = t;
    ctl->R = alive[t];
    ctl->pos = t * ctl->k;
  }
  cudaGraphSetConditional(handle, more ? 1u : 0u);
}

// Same step advance for the unrolled (plain) loop graphs: the host launches
// exactly the segment's step count, so no loop condition is set.
// Once every row (sentence, in beam mode) has finished, R drops to 0 and the
// remaining captured steps' kernels return immediately. Greedy (done != nullptr):
// rows finish at their own natural EOS (decoding.py:149-150), so the live count is
// 1 + the last unfinished row below the cap-predicted one (rows are cap-sorted;
// every row past it has finished) -- the batch shrinks with the finished tail
// instead of with the caps. ctl->pad accumulates the rows computed (statistics).
// (one block; c = the control block as it stands after this step's selection)
__device__ __forceinline__ void stage1_advance_block(StepCtl* ctl, const StepCtl& c, const int* __restrict__ alive,
                                                     const int* __restrict__ done, int* s_last) {
  const int t = c.t + 1;
  const bool more = c.finished < c.nrows && t < c.max_cap && alive[t] > 0;
  int R = more ? alive[t] : 0;
  if (done != nullptr && more) {  // (block-uniform branch)
    int last = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x)
      if (!__ldcg(done + r)) last = r + 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (blockDim.x > 32) {  // small buckets launch one warp: no block barrier on the step's critical path
      if (threadIdx.x == 0) *s_last = 0;
      __syncthreads();
      if ((threadIdx.x & 31) == 0 && last > 0) atomicMax(s_last, last);
      __syncthreads();
      last = *s_last;
    }
    R = last;
  }
  if (threadIdx.x == 0) {
    if (c.finished >= c.nrows) {
      ctl->R = 0;
    } else if (more) {
      ctl->t = t;
      ctl->R = R;
      ctl->pos = t * c.k;
      ctl->pad = c.pad + R;
    }
  }
}

__global__ void stage1_advance_plain_kernel(StepCtl* ctl, const int* __restrict__ alive, const int* __restrict__ done) {
  pdl_enter();
  __shared__ int s_last;
  const StepCtl c = *ctl;
  stage1_advance_block(ctl, c, alive, done, &s_last);
}

// Single-CTA row buckets (<= 4 greedy rows, one warp per row, plain loop
// graphs): the selection and the step advance in one launch. The CTA knows
// every row's new done flag and the step's finishes itself, and alive[t + 1]
// is requested with the partials, so the advance (stage1_advance_plain_kernel's
// rule) costs no extra memory round trip; it is decided before the embedding.
template <typename T>
__global__ void greedy_select_advance_kernel(VocabParts parts, GreedyState st, int R, StepCtl* ctl,
                                             const int* __restrict__ alive) {
  pdl_enter();
  __shared__ int s_done[4], s_fin[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rr = min(warp, R - 1);
  const StepCtl c = *ctl;
  const int done_v = st.done[rr];
  const int al = alive[c.t + 1];  // (alive holds max_cap + 1 entries)
  const RowStat rs = merge_row1(parts, rr);
  int tok = 0, fin = 0;
  const bool live = warp < c.R;
  if (live) tok = greedy_pick_row(rs, st, warp, c.t, done_v, ctl, &fin);
  if (lane == 0) {
    s_done[warp] = (warp < R && !live) ? done_v : (live ? (done_v | fin) : 1);
    s_fin[warp] = fin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int finished = c.finished;
    for (int r = 0; r < 4; ++r) finished += s_fin[r];
    const int t = c.t + 1;
    const bool more = finished < c.nrows && t < c.max_cap && al > 0;
    if (finished >= c.nrows) {
      ctl->R = 0;
    } else if (more) {
      int last = 0;  // 1 + the last unfinished row below the cap-predicted count
      for (int r = 0; r < min(al, 4); ++r)
        if (!s_done[r]) last = r + 1;
      ctl->t = t;
      ctl->R = last;
      ctl->pos = t * c.k;
      ctl->pad = c.pad + last;
    }
  }
  if (live) greedy_embed_row<T>(st, warp, c.t, c.k, tok);
}

// Final per-row stats (protocol face / Stage II): amax + renormalised logprob.
template <int KT>
__global__ void rowstat_kernel(VocabParts parts, int R, int kt, RowStat* __restrict__ out,
                               const int* __restrict__ R_dev = nullptr) {
  pdl_enter();
  if (R_dev) R = *R_dev;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= R) return;
  const RowStat rs = (KT == 1 && kt == 1) ? merge_row1(parts, row) : merge_row<KT>(parts, row, kt);
  if ((threadIdx.x & 31) == 0) out[row] = rs;
}

// ---------------------------------------------------------------------------
// Stage-II input (decoding.py:208-217, :268-276): candidate c (sentence
// cand_sent[c]) with m anchors gets slot rows [off[c], off[c] + slot[c]):
// position j < k*m holds MASK, or the anchor z_{(j+1)/k-1} when (j+1) % k == 0;
// positions are j + 1. Rows past k*m are padding (never attended, ignored).
// ---------------------------------------------------------------------------
// Stage-II candidates: anchors of candidate c live at tok + (tok_off ?
// tok_off[c] : c * cap), len[c] anchors (0 = no such candidate).
struct Stage2Cands {
  const int* tok;
  const int* tok_off;
  int cap;
  const int* len;
  const double* s_at;  // [C] Stage-I score of the candidate
  const int* forced;   // [C]
  const int* steps;    // [S] Stage-I steps of the sentence
};

__global__ void stage2_build_kernel(Stage2Cands cands, const int* __restrict__ off, const int* __restrict__ slot, int C,
                                    int k, int* __restrict__ ids, int* __restrict__ pos, int* __restrict__ qlen) {
  pdl_enter();
  const int c = blockIdx.x;
  if (c >= C) return;
  const int m = cands.len[c];
  const int T = k * m;
  const int sl = slot[c], o = off[c];
  const int* z = cands.tok + (cands.tok_off ? (size_t)cands.tok_off[c] : (size_t)c * cands.cap);
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

// AT baseline result (decoding.py:173-185, beam 1): the finished hypothesis'
// tokens up to its EOS, score s / len^alpha with len counting the EOS,
// decoder_calls = Stage-I steps. One warp per sentence.
__global__ void at_finish_kernel(Stage2Cands cands, float alpha, int max_len, int S, Stage2Out out) {
  pdl_enter();
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  const int m = cands.len[s];  // generated tokens including EOS (= steps for greedy)
  const int* tok = cands.tok + (size_t)s * cands.cap;
  int first_eos = m;
  for (int j0 = 0; j0 < m; j0 += 32) {
    const int j = j0 + lane;
    const unsigned ball = __ballot_sync(0xffffffffu, j < m && tok[j] == EOS_ID);
    if (ball) {
      first_eos = j0 + __ffs(ball) - 1;
      break;
    }
  }
  const int n = min(first_eos, max_len);
  const int dst = out.out_index ? out.out_index[s] : s;
  for (int j = lane; j < n; j += 32) out.tokens[(size_t)dst * max_len + j] = tok[j];
  if (lane == 0) {
    const double sat = cands.s_at[s];
    out.lens[dst] = n;
    out.scores[(size_t)dst * 3 + 0] = sat;
    out.scores[(size_t)dst * 3 + 1] = 0.0;
    out.scores[(size_t)dst * 3 + 2] = sat / pow((double)max(m, 1), (double)alpha);
    out.calls[dst] = cands.steps[s];
    out.forced[dst] = (unsigned char)cands.forced[s];
  }
}

__global__ void stage2_finish_kernel(const int* __restrict__ ids, const int* __restrict__ off,
                                     const int* __restrict__ qlen, const int* __restrict__ mrow_off,
                                     const RowStat* __restrict__ mstat, const int* __restrict__ cand_beg,
                                     Stage2Cands cands, int k, float alpha, int max_len, int S, Stage2Out out) {
  pdl_enter();
  const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  int best = -1;
  double best_score = 0.0, best_cmlm = 0.0;
  for (int c = cand_beg[s]; c < cand_beg[s + 1]; ++c) {
    const int T = qlen[c];
    if (T == 0) continue;  // no such candidate
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
    const double sc = (cands.s_at[c] + cmlm) / pow((double)T, (double)alpha);
    if (best < 0 || sc > best_score) {
      best = c;
      best_score = sc;
      best_cmlm = cmlm;
    }
  }
  const int dst = out.out_index ? out.out_index[s] : s;
  if (best < 0) {  // no finished hypothesis reached Stage II (cannot happen with a step cap)
    if (lane == 0) {
      out.lens[dst] = 0;
      out.scores[(size_t)dst * 3 + 0] = out.scores[(size_t)dst * 3 + 1] = out.scores[(size_t)dst * 3 + 2] = 0.0;
      out.calls[dst] = cands.steps[s] + 1;
      out.forced[dst] = 0;
    }
    return;
  }
  const int c = best;
  const int T = qlen[c];
  const int o = off[c];
  const int mo = mrow_off[c];
  // first EOS in the filled sequence (warp scan over positions)
  int first_eos = T;
  for (int j0 = 0; j0 < T; j0 += 32) {
    const int j = j0 + lane;
    int tok = -1;
    if (j < T) {
      tok = ((j + 1) % k != 0) ? mstat[mo + j - (j + 1) / k].id[0] : ids[o + j];
      if (tok == 0x7fffffff) tok = EOS_ID;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, j < T && tok == EOS_ID);
    if (ball) {
      first_eos = j0 + __ffs(ball) - 1;
      break;
    }
  }
  const int n = min(first_eos, max_len);
  for (int j = lane; j < n; j += 32) {
    int tok = ((j + 1) % k != 0) ? mstat[mo + j - (j + 1) / k].id[0] : ids[o + j];
    if (tok == 0x7fffffff) tok = EOS_ID;
    out.tokens[(size_t)dst * max_len + j] = tok;
  }
  if (lane == 0) {
    out.lens[dst] = n;
    out.scores[(size_t)dst * 3 + 0] = cands.s_at[c];
    out.scores[(size_t)dst * 3 + 1] = best_cmlm;
    out.scores[(size_t)dst * 3 + 2] = best_score;
    out.calls[dst] = cands.steps[s] + 1;
    out.forced[dst] = (unsigned char)cands.forced[c];
  }
}

// ---------------------------------------------------------------------------
// Stage-I beam search on device (decoding.py:90-155, b_at > 1).
// Sentence s owns rows [s*beam, (s+1)*beam); row s*beam + h holds live
// hypothesis h. One warp per sentence per step:
//   1. candidates: every live hypothesis contributes its top (beam+1)
//      generable tokens (or EOS at the cap), score += fp32 log-prob in fp64;
//   2. stable sort by (-score, token) -- warp-parallel rank counting with the
//      generation index as the final tie break (Python's stable sort);
//   3. lane 0 applies the acceptance rules: EOS finishes if rank < beam or
//      greedy; others fill new_live up to beam; greedy-chain reservation;
//      break when nothing is live or (>= beam finished and greedy done);
//   4. the warp reorders the rows (anchor history + KV history index map,
//      ping-pong buffers by step parity) and embeds the next step's inputs.
// Finished hypotheses: a per-sentence top-b_nat list (stable by -score) plus
// the greedy one, in a (b_nat + 2)-slot token pool.
// ---------------------------------------------------------------------------
constexpr int BEAM_MAX = 7, BEAM_MAXC = BEAM_MAX * (BEAM_MAX + 1);

struct BeamState {
  int beam, bnat, cap;
  int* feed;         // [rows]
  double* score;     // [rows]
  int* greedy;       // [rows]
  int* anchors[2];   // [rows][cap] ping-pong
  int* hist[2];      // [rows][cap] ping-pong
  int* live_n;       // [S]
  int* done;         // [S]
  int* nsteps;       // [S]
  int* n_fin;        // [S]
  int* greedy_done;  // [S]
  const int* caps;   // [S]
  // finished store, F = bnat + 2 slots per sentence
  int* f_count;      // [S] entries in the top list
  int* f_list;       // [S][bnat] slot of the i-th best
  int* f_gslot;      // [S] slot of the finished greedy hypothesis (-1: none)
  double* f_score;   // [S][F]
  int* f_len;        // [S][F]
  int* f_forced;     // [S][F]
  int* f_tok;        // [S][F][cap]
  // next-step embedding
  const void* E;
  const float* pe;
  const float* ln_g;
  const float* ln_b;
  float* x;
  void* y;
  float scale;
  int d;
};

__global__ void beam_init_kernel(BeamState st, int S, int bos) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = S * st.beam;
  if (i < rows) {
    st.feed[i] = bos;
    st.score[i] = 0.0;
    st.greedy[i] = (i % st.beam) == 0;
    for (int j = 0; j < st.cap; ++j) st.hist[0][(size_t)i * st.cap + j] = i;
  }
  if (i < S) {
    st.live_n[i] = 1;
    st.done[i] = 0;
    st.nsteps[i] = 0;
    st.n_fin[i] = 0;
    st.greedy_done[i] = 0;
    st.f_count[i] = 0;
    st.f_gslot[i] = -1;
  }
}

// grid = sentences (upper bound), block = 32 * BEAM_MAX threads: warp 0 runs
// the selection, then warp j embeds row j of the sentence for the next step.
template <typename T>
__global__ void __launch_bounds__(32 * BEAM_MAX) beam_select_kernel(const RowStat* __restrict__ rs, BeamState st,
                                                                   int S, int t, int k, StepCtl* ctl) {
  pdl_enter();
  __shared__ double cs[1][BEAM_MAXC];
  __shared__ int ct[1][BEAM_MAXC], cp[1][BEAM_MAXC], cg[1][BEAM_MAXC], ord[1][BEAM_MAXC];
  __shared__ int nl_s[1], brk_s[1], ntok[1][BEAM_MAX], npar[1][BEAM_MAX], ncopy[1], copy_slot[1][BEAM_MAXC],
      copy_src[1][BEAM_MAXC];
  const int beam = st.beam;
  if (ctl) {
    S = ctl->R / beam;
    t = ctl->t;
    k = ctl->k;
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = 0;
  const int s = blockIdx.x;
  if (s >= S) return;
  const int r0 = s * beam;
  const int cur = t & 1, nxt = cur ^ 1;
  const int cap = st.cap;
  const int F = st.bnat + 2;
  if (wid == 0 && !st.done[s]) {
    const int L = st.live_n[s];
    const bool last = (t == st.caps[s] - 1);
    const int nt = last ? 1 : beam + 1;
    const int n = L * nt;
    // 1. candidates in generation order (parent-major, then rank in the row's top list)
    for (int i = lane; i < n; i += 32) {
      const int h = i / nt, q = i - h * nt;
      const RowStat& R = rs[r0 + h];
      int g = R.id[0];
      if (g == 0x7fffffff) g = EOS_ID;
      int tok;
      float logit;
      if (last) {
        tok = EOS_ID;
        logit = R.eos;
      } else {
        tok = R.id[q];
        logit = R.val[q];
        if (tok == 0x7fffffff) {  // fewer generable ids than beam + 1: never selectable
          tok = EOS_ID;
          logit = -INFINITY;
        }
      }
      const float lp = (logit - R.mx) - R.lse;
      cs[w][i] = st.score[r0 + h] + (double)lp;
      ct[w][i] = tok;
      cp[w][i] = h;
      cg[w][i] = st.greedy[r0 + h] && (last || tok == g);
    }
    __syncwarp();
    // 2. stable rank by (-score, token, generation index)
    for (int i = lane; i < n; i += 32) {
      const double si = cs[w][i];
      const int ti = ct[w][i];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double sj = cs[w][j];
        const int tj = ct[w][j];
        rank += (sj > si) || (sj == si && (tj < ti || (tj == ti && j < i)));
      }
      ord[w][rank] = i;
    }
    __syncwarp();
    // 3. acceptance rules (lane 0, sequential in rank order)
    if (lane == 0) {
      int nl = 0, nc = 0;
      bool gdone = st.greedy_done[s] != 0;
      int* flist = st.f_list + (size_t)s * st.bnat;
      auto finish = [&](int i) {
        const bool g = cg[w][i] != 0;
        st.n_fin[s] += 1;
        const double sc = cs[w][i];
        // stable insert position in the top-b_nat list (after equal scores)
        int cnt = st.f_count[s];
        int p = cnt;
        for (int a = 0; a < cnt; ++a)
          if (st.f_score[(size_t)s * F + flist[a]] < sc) {
            p = a;
            break;
          }
        const bool top = p < st.bnat;
        if (!top && !g) return;
        // free slot: referenced neither by the top list nor by the greedy pointer
        int slot = -1;
        for (int q = 0; q < F && slot < 0; ++q) {
          bool used = (st.f_gslot[s] == q);
          for (int a = 0; a < cnt && !used; ++a) used = flist[a] == q;
          if (!used) slot = q;
        }
        st.f_score[(size_t)s * F + slot] = sc;
        st.f_len[(size_t)s * F + slot] = t + 1;
        st.f_forced[(size_t)s * F + slot] = last ? 1 : 0;
        copy_slot[w][nc] = slot;
        copy_src[w][nc] = r0 + cp[w][i];
        ++nc;
        if (top) {
          const int newcnt = cnt < st.bnat ? cnt + 1 : st.bnat;
          for (int a = newcnt - 1; a > p; --a) flist[a] = flist[a - 1];
          flist[p] = slot;
          st.f_count[s] = newcnt;
        }
        if (g) {
          st.f_gslot[s] = slot;
          gdone = true;
        }
      };
      for (int rank = 0; rank < n; ++rank) {
        const int i = ord[w][rank];
        if (ct[w][i] == EOS_ID) {
          if (rank < beam || cg[w][i]) finish(i);
        } else if (nl < beam) {
          ntok[w][nl] = i;
          ++nl;
        }
      }
      if (!gdone) {
        bool any = false;
        for (int a = 0; a < nl; ++a) any |= cg[w][ntok[w][a]] != 0;
        if (!any && nl > 0) {
          for (int rank = 0; rank < n; ++rank) {
            const int i = ord[w][rank];
            if (cg[w][i] && ct[w][i] != EOS_ID) {
              ntok[w][nl - 1] = i;
              break;
            }
          }
        }
      }
      st.greedy_done[s] = gdone;
      const bool brk = nl == 0 || (st.n_fin[s] >= beam && gdone);
      if (brk) {
        st.done[s] = 1;
        st.nsteps[s] = t + 1;
        if (ctl) atomicAdd(&ctl->finished, 1);
      }
      for (int a = 0; a < nl; ++a) npar[w][a] = cp[w][ntok[w][a]];
      nl_s[w] = nl;
      brk_s[w] = brk;
      ncopy[w] = nc;
    }
    __syncwarp();
    // finished token copies: parent history + EOS
    for (int c = 0; c < ncopy[w]; ++c) {
      int* dst = st.f_tok + ((size_t)s * F + copy_slot[w][c]) * cap;
      const int* src = st.anchors[cur] + (size_t)copy_src[w][c] * cap;
      for (int j = lane; j <= t; j += 32) dst[j] = (j < t) ? src[j] : EOS_ID;
    }
    // 4. reorder into the next buffers (rows past nl continue from row 0, decoding.py:151)
    if (!brk_s[w]) {
      const int nl = nl_s[w];
      for (int j = 0; j < beam; ++j) {
        const int par = j < nl ? npar[w][j] : 0;
        const int src = r0 + par, dst = r0 + j;
        const int* ah = st.anchors[cur] + (size_t)src * cap;
        int* an = st.anchors[nxt] + (size_t)dst * cap;
        const int* hh = st.hist[cur] + (size_t)src * cap;
        int* hn = st.hist[nxt] + (size_t)dst * cap;
        const int tok = j < nl ? ct[w][ntok[w][j]] : st.feed[dst];
        for (int q = lane; q <= t; q += 32) {
          an[q] = (q < t) ? ah[q] : tok;
          hn[q] = (q < t) ? hh[q] : src;  // slot t was appended by physical row src
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (int j = 0; j < nl; ++j) {
          const int i = ntok[w][j];
          st.score[r0 + j] = cs[w][i];
          st.greedy[r0 + j] = cg[w][i];
          st.feed[r0 + j] = ct[w][i];
        }
        for (int j = nl; j < beam; ++j) st.greedy[r0 + j] = 0;
        st.live_n[s] = nl;
      }
    }
  }
  __syncthreads();
  // next step's embedding, one warp per row (finished rows feed stale tokens)
  if (st.x != nullptr && wid < beam) {
    const int r = r0 + wid;
    const int tok = st.feed[r];
    warp_embed_ln<T>(static_cast<const T*>(st.E), st.pe, st.ln_g, st.ln_b, st.scale, st.d, tok, (t + 1) * k,
                     st.x + (size_t)r * st.d, static_cast<T*>(st.y) + (size_t)r * st.d);
  }
}

// Stage-II candidates of every sentence (decoding.py:262-266): the top-b_nat
// finished hypotheses by score (stable), the greedy one forced into the last
// place when missing. Candidate c = s * b_nat + i.
__global__ void beam_candidates_kernel(BeamState st, int S, int* __restrict__ c_off, int* __restrict__ c_len,
                                       double* __restrict__ c_sat, int* __restrict__ c_forced) {
  pdl_enter();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const int F = st.bnat + 2;
  const int* flist = st.f_list + (size_t)s * st.bnat;
  int cnt = st.f_count[s];
  int sl[8];
  for (int a = 0; a < cnt; ++a) sl[a] = flist[a];
  const int g = st.f_gslot[s];
  if (g >= 0 && cnt > 0) {
    bool in = false;
    for (int a = 0; a < cnt; ++a) in |= sl[a] == g;
    if (!in) sl[cnt - 1] = g;
  } else if (g >= 0 && cnt == 0) {
    sl[0] = g;
    cnt = 1;
  }
  for (int a = 0; a < st.bnat; ++a) {
    const int c = s * st.bnat + a;
    if (a < cnt) {
      const int slot = sl[a];
      c_off[c] = (s * F + slot) * st.cap;
      c_len[c] = st.f_len[(size_t)s * F + slot];
      c_sat[c] = st.f_score[(size_t)s * F + slot];
      c_forced[c] = st.f_forced[(size_t)s * F + slot];
    } else {
      c_off[c] = 0;
      c_len[c] = 0;
      c_sat[c] = 0.0;
      c_forced[c] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// small utility kernels
// ---------------------------------------------------------------------------
// packed gather of sentences into a new order: dst sentence i <- src sentence perm[i]
__global__ void gather_sentences_kernel(const int* __restrict__ src, const int* __restrict__ src_off,
                                        const int* __restrict__ dst_off, const int* __restrict__ perm,
                                        int* __restrict__ dst, int* __restrict__ pos, int n, int vocab) {
  pdl_enter();
  const int i = blockIdx.x;
  if (i >= n) return;
  const int p = perm[i];
  // sources longer than max_len keep their first dst_off[i + 1] - dst_off[i]
  // tokens (decoding.py:260 truncation); the raw offsets still step over the full source
  const int so = src_off[p], d0 = dst_off[i], len = min(src_off[p + 1] - so, dst_off[i + 1] - d0);
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    const int id = src[so + j];
    dst[d0 + j] = (id >= 0 && id < vocab) ? id : EOS_ID;  // device ids are not validated on the host
    pos[d0 + j] = j;
  }
}

// Stage-I row initialisation: feed = bos, history slot map = identity.
// Debug (option "debug_spin"): occupy the stream for `ns` nanoseconds so the
// host runs ahead; phase times measured behind it are pure device time.
__global__ void debug_spin_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t1 = t0;
  while (t1 - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
}

__global__ void stage1_init_kernel(int R, int cap, int bos, int* feed, int* done, int* nsteps, int* forced,
                                   double* score, int* hist) {
  pdl_enter();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  feed[r] = bos;
  done[r] = 0;
  nsteps[r] = 0;
  forced[r] = 0;
  score[r] = 0.0;
  for (int j = 0; j < cap; ++j) hist[(size_t)r * cap + j] = r;
}

// Stage-I row -> encoded sentence (beam rows share their sentence's memory)
// Rows past the live ones (up to the graph's row bucket) name sentence B,
// whose source length in the header is 0: the cross-attention K/V prefetch,
// which runs before the row count resolves, then reads nothing.
__global__ void rowseq_fill_kernel(int* __restrict__ rowseq, int rows, int rows_cap, int beam, int n_seq) {
  pdl_enter();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows_cap) rowseq[r] = r < rows ? r / beam : n_seq;
}

// Beam reorder as an index permutation (infer.py:307-318): row j continues
// from old row parents[j]; history slots 0..t-1 follow the parent.
__global__ void reorder_hist_kernel(const int* __restrict__ parents, const int* __restrict__ hist_in,
                                    int* __restrict__ hist_out, int R, int cap, int t) {
  pdl_enter();
  const int r = blockIdx.x;
  if (r >= R) return;
  const int p = parents[r];
  for (int j = threadIdx.x; j < cap; j += blockDim.x)
    hist_out[(size_t)r * cap + j] = (j < t) ? hist_in[(size_t)p * cap + j] : r;
}

// Full-row log-softmax in place (protocol-face step(), infer.py:296-301).
__global__ void logsoftmax_rows_kernel(float* __restrict__ l, int ld, int V) {
  pdl_enter();
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
  pdl_enter();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = __float2bfloat16_rn(a[i]);
}

}  // namespace hrt
