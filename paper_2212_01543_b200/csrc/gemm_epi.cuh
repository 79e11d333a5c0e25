// GEMM epilogue functors shared by the tcgen05 GEMM (bf16) and the SIMT GEMM
// (fp32). Protocol: State; begin(st,row,n0); chunk(st,row,col0,v,n); end(st,row,n0).
//   EpiBias       y = acc + b           (QKV / Q / cross-KV projections, infer.py:169-172)
//   EpiBiasRelu   y = relu(acc + b)     (FFN1, infer.py:207-209)
//   EpiResidual   x += acc + b          (O-proj / FFN2 + residual, infer.py:204-205, :210-212)
//   EpiStoreF32   logits = acc          (parity / debug logits)
#pragma once
#include "common.cuh"

namespace hrt {

template <typename T>
__device__ __forceinline__ void store_row_chunk(T* dst, const float* v, int n);

template <>
__device__ __forceinline__ void store_row_chunk<float>(float* dst, const float* v, int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else {
    for (int i = 0; i < n; ++i) dst[i] = v[i];
  }
}

template <>
__device__ __forceinline__ void store_row_chunk<bf16>(bf16* dst, const float* v, int n) {
  if (n == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 u;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i + 0], v[i + 1]);
      __nv_bfloat162 p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]);
      __nv_bfloat162 p3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      u.z = *reinterpret_cast<uint32_t*>(&p2);
      u.w = *reinterpret_cast<uint32_t*>(&p3);
      *reinterpret_cast<uint4*>(dst + i) = u;
    }
  } else {
    for (int i = 0; i < n; ++i) dst[i] = __float2bfloat16_rn(v[i]);
  }
}

template <typename T, bool RELU>
struct EpiBiasT {
  T* out;
  int ldo;
  const float* bias;
  struct State {};
  __device__ __forceinline__ void begin(State&, int, int) const {}
  __device__ __forceinline__ void chunk(State&, int row, int col0, const float* v, int n) const {
    float w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < n) {
        float a = v[i] + bias[col0 + i];
        w[i] = RELU ? fmaxf(a, 0.f) : a;
      }
    }
    store_row_chunk<T>(out + (size_t)row * ldo + col0, w, n);
  }
  __device__ __forceinline__ void end(State&, int, int) const {}
};

struct EpiResidual {
  float* x;
  int ldx;
  const float* bias;
  struct State {};
  __device__ __forceinline__ void begin(State&, int, int) const {}
  __device__ __forceinline__ void chunk(State&, int row, int col0, const float* v, int n) const {
    float* p = x + (size_t)row * ldx + col0;
    if (n == 32 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 a = *reinterpret_cast<float4*>(p + i);
        a.x += v[i] + bias[col0 + i];
        a.y += v[i + 1] + bias[col0 + i + 1];
        a.z += v[i + 2] + bias[col0 + i + 2];
        a.w += v[i + 3] + bias[col0 + i + 3];
        *reinterpret_cast<float4*>(p + i) = a;
      }
    } else {
      for (int i = 0; i < n; ++i) p[i] += v[i] + bias[col0 + i];
    }
  }
  __device__ __forceinline__ void end(State&, int, int) const {}
};

struct EpiStoreF32 {
  float* out;
  int ldo;
  struct State {};
  __device__ __forceinline__ void begin(State&, int, int) const {}
  __device__ __forceinline__ void chunk(State&, int row, int col0, const float* v, int n) const {
    store_row_chunk<float>(out + (size_t)row * ldo + col0, v, n);
  }
  __device__ __forceinline__ void end(State&, int, int) const {}
};

}  // namespace hrt
