// Element-wise GEMM epilogue functors shared by the tcgen05 GEMM (bf16) and
// the SIMT GEMM (fp32). apply4 handles 4 consecutive columns (16 B aligned),
// apply1 a single element (SIMT edge tiles).
//   EpiBiasT<T,false>  y = acc + b           (QKV / Q / cross-KV projections, infer.py:169-172)
//   EpiBiasT<T,true>   y = relu(acc + b)     (FFN1, infer.py:207-209)
//   EpiResidual        x += acc + b          (O-proj / FFN2 + residual, infer.py:204-205, :210-212)
//   EpiStoreF32        logits = acc          (parity / debug logits)
#pragma once
#include <type_traits>

#include "common.cuh"

namespace hrt {

__device__ __forceinline__ void store4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void store4(bf16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
  __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

template <typename T, bool RELU>
struct EpiBiasT {
  static constexpr bool kRowWise = false;
  T* out;
  int ldo;
  const float* bias;
  __host__ __device__ int ld() const { return ldo; }
  __device__ __forceinline__ void apply4(int row, int col, float4 v) const {
    const float4 b = *reinterpret_cast<const float4*>(bias + col);
    v.x += b.x;
    v.y += b.y;
    v.z += b.z;
    v.w += b.w;
    if (RELU) {
      v.x = fmaxf(v.x, 0.f);
      v.y = fmaxf(v.y, 0.f);
      v.z = fmaxf(v.z, 0.f);
      v.w = fmaxf(v.w, 0.f);
    }
    store4(out + (size_t)row * ldo + col, v);
  }
  __device__ __forceinline__ void apply8(int row0, int col, const float4* v, int M) const {
    const float4 b = *reinterpret_cast<const float4*>(bias + col);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = row0 + 4 * i;
      if (row < M) {
        float4 a = v[i];
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
        if (RELU) {
          a.x = fmaxf(a.x, 0.f);
          a.y = fmaxf(a.y, 0.f);
          a.z = fmaxf(a.z, 0.f);
          a.w = fmaxf(a.w, 0.f);
        }
        store4(out + (size_t)row * ldo + col, a);
      }
    }
  }
  __device__ __forceinline__ void apply1(int row, int col, float v) const {
    float a = v + bias[col];
    if (RELU) a = fmaxf(a, 0.f);
    out[(size_t)row * ldo + col] = from_f<T>(a);
  }
  // TMA-store form (tcgen05 epilogue, bf16 out): one row's 32 columns -> 16 packed bf16 pairs.
  // bias_lane = bias[col0 + lane] (one coalesced load per chunk, requested a chunk ahead);
  // column j's bias is broadcast from lane j by a shuffle
  static constexpr bool kTmaStore = std::is_same<T, bf16>::value;
  __device__ __forceinline__ float bias_of(int col) const { return __ldg(bias + col); }
  __device__ __forceinline__ void row32_pack_shfl(float bias_lane, const float* v, uint32_t* pk) const {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float a0 = v[2 * j] + __shfl_sync(0xffffffffu, bias_lane, 2 * j);
      float a1 = v[2 * j + 1] + __shfl_sync(0xffffffffu, bias_lane, 2 * j + 1);
      if (RELU) {
        a0 = fmaxf(a0, 0.f);
        a1 = fmaxf(a1, 0.f);
      }
      __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
      pk[j] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  __device__ __forceinline__ void row32_pack(int col0, const float* v, uint32_t* pk) const {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col0) + j);
      float a0 = v[4 * j] + b.x, a1 = v[4 * j + 1] + b.y, a2 = v[4 * j + 2] + b.z, a3 = v[4 * j + 3] + b.w;
      if (RELU) {
        a0 = fmaxf(a0, 0.f);
        a1 = fmaxf(a1, 0.f);
        a2 = fmaxf(a2, 0.f);
        a3 = fmaxf(a3, 0.f);
      }
      __nv_bfloat162 lo = __floats2bfloat162_rn(a0, a1), hi = __floats2bfloat162_rn(a2, a3);
      pk[2 * j] = *reinterpret_cast<uint32_t*>(&lo);
      pk[2 * j + 1] = *reinterpret_cast<uint32_t*>(&hi);
    }
  }
  // split form for latency-bound callers: every operand load issued before any store
  __device__ __forceinline__ float2 load2(int, int col) const { return make_float2(__ldg(bias + col), 0.f); }
  __device__ __forceinline__ void store2(int row, int col, float v, float2 pre) const {
    float a = v + pre.x;
    if (RELU) a = fmaxf(a, 0.f);
    out[(size_t)row * ldo + col] = from_f<T>(a);
  }
};

struct EpiResidual {
  static constexpr bool kRowWise = false;
  float* x;
  int ldx;
  const float* bias;
  // tcgen05 epilogue only: x += acc + bias as fire-and-forget L2 reductions
  // (red.global.add.v4.f32) instead of a prefetched read-modify-write. One add per
  // element, so the result is the same bits as the load / add / store form.
  bool red = false;
  __host__ __device__ int ld() const { return ldx; }
  __device__ __forceinline__ void apply4(int row, int col, float4 v) const {
    float* p = x + (size_t)row * ldx + col;
    const float4 b = *reinterpret_cast<const float4*>(bias + col);
    float4 a = *reinterpret_cast<float4*>(p);
    a.x += v.x + b.x;
    a.y += v.y + b.y;
    a.z += v.z + b.z;
    a.w += v.w + b.w;
    *reinterpret_cast<float4*>(p) = a;
  }
  __device__ __forceinline__ void apply8(int row0, int col, const float4* v, int M) const {
    const float4 b = *reinterpret_cast<const float4*>(bias + col);
    float4 prev[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (row0 + 4 * i < M) prev[i] = *reinterpret_cast<const float4*>(x + (size_t)(row0 + 4 * i) * ldx + col);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (row0 + 4 * i < M) {
        float4 a = prev[i];
        a.x += v[i].x + b.x;
        a.y += v[i].y + b.y;
        a.z += v[i].z + b.z;
        a.w += v[i].w + b.w;
        *reinterpret_cast<float4*>(x + (size_t)(row0 + 4 * i) * ldx + col) = a;
      }
    }
  }
  // prefetching form (tcgen05 epilogue): the residual rows of a 32-column chunk are
  // requested one chunk ahead, so their DRAM latency overlaps the previous chunk
  static constexpr bool kPrefetch = true;
  __device__ __forceinline__ void prefetch8(int row0, int col, int M, float4 (&p)[8]) const {
    if (red) return;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      p[i] = row0 + 4 * i < M ? *reinterpret_cast<const float4*>(x + (size_t)(row0 + 4 * i) * ldx + col)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ void apply8_pre(int row0, int col, const float4* v, int M, const float4 (&prev)[8]) const {
    const float4 b = *reinterpret_cast<const float4*>(bias + col);
    if (red) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (row0 + 4 * i < M)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(x + (size_t)(row0 + 4 * i) * ldx + col),
                       "f"(v[i].x + b.x), "f"(v[i].y + b.y), "f"(v[i].z + b.z), "f"(v[i].w + b.w)
                       : "memory");
      return;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (row0 + 4 * i < M) {
        float4 a = prev[i];
        a.x += v[i].x + b.x;
        a.y += v[i].y + b.y;
        a.z += v[i].z + b.z;
        a.w += v[i].w + b.w;
        *reinterpret_cast<float4*>(x + (size_t)(row0 + 4 * i) * ldx + col) = a;
      }
    }
  }
  __device__ __forceinline__ void apply1(int row, int col, float v) const {
    x[(size_t)row * ldx + col] += v + bias[col];
  }
  __device__ __forceinline__ float2 load2(int row, int col) const {
    return make_float2(x[(size_t)row * ldx + col], __ldg(bias + col));
  }
  __device__ __forceinline__ void store2(int row, int col, float v, float2 pre) const {
    x[(size_t)row * ldx + col] = pre.x + (v + pre.y);
  }
};

struct EpiStoreF32 {
  static constexpr bool kRowWise = false;
  float* out;
  int ldo;
  __host__ __device__ int ld() const { return ldo; }
  __device__ __forceinline__ void apply4(int row, int col, float4 v) const {
    store4(out + (size_t)row * ldo + col, v);
  }
  __device__ __forceinline__ void apply8(int row0, int col, const float4* v, int M) const {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (row0 + 4 * i < M) store4(out + (size_t)(row0 + 4 * i) * ldo + col, v[i]);
  }
  __device__ __forceinline__ void apply1(int row, int col, float v) const { out[(size_t)row * ldo + col] = v; }
  __device__ __forceinline__ float2 load2(int, int) const { return make_float2(0.f, 0.f); }
  __device__ __forceinline__ void store2(int row, int col, float v, float2) const { out[(size_t)row * ldo + col] = v; }
};

}  // namespace hrt
