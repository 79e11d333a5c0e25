// fp32 SIMT GEMM  C[M, N] = A[M, K] . B[N, K]^T  for the fp32 (config-1 parity)
// path. kind::tf32 tensor cores would truncate operands to 10 mantissa bits,
// which the 1e-3 fp32 logits bound does not leave room for (SURVEY §7 hard
// part 3), so fp32 runs on FFMA: 64x64 tiles, BK=16, 4x4 per thread, any
// M/N/K (no alignment requirements: toy configs with d=16 use it too).
#pragma once
#include "common.cuh"

namespace hrt {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16, SG_THREADS = 256;

template <typename T, class Epi>
__global__ void __launch_bounds__(SG_THREADS) simt_gemm_kernel(const T* __restrict__ A, int lda,
                                                               const T* __restrict__ B, int ldb, int M, int N,
                                                               int K, const int* __restrict__ M_dev, Epi epi, int aligned4) {
  pdl_enter();
  if (M_dev) M = *M_dev;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  if (m0 >= M) return;
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int lr = tid >> 2, lc = (tid & 3) * 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += SG_BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = k0 + lc + i;
      const int am = m0 + lr, bn = n0 + lr;
      As[lc + i][lr] = (am < M && kk < K) ? to_f(A[(size_t)am * lda + kk]) : 0.f;
      Bs[lc + i][lr] = (bn < N && kk < K) ? to_f(B[(size_t)bn * ldb + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        b[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    const int col = n0 + tx * 4;
    if (row < M && col < N) {
      if (col + 4 <= N && ((size_t)col & 3) == 0 && aligned4) {
        epi.apply4(row, col, make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
      } else {
        for (int j = 0; j < 4 && col + j < N; ++j) epi.apply1(row, col + j, acc[i][j]);
      }
    }
  }
}

}  // namespace hrt

namespace hrt {

// fp32 GEMV for the latency-bound shapes (up to GF_MAXM * gridDim.y rows:
// decode steps, batch-1 encoder / Stage II / vocabulary of the fp32 parity
// path). One warp per output feature over the full K: lane l reads
// W[n][k..k+3] for k = 4 l + 128 i as float4 (coalesced 512-byte rows), FFMA
// against GF_MAXM activation rows (blockIdx.y picks the row block; the weight
// re-reads of further blocks hit L2), then a fixed-order warp reduction
// (deterministic). Weights are requested before the PDL grid-dependency wait.
constexpr int GF_WARPS = 16, GF_MAXM = 8;

template <int KI, class Epi>  // KI: K / 128 (float4 chunks per lane)
__global__ void __launch_bounds__(GF_WARPS * 32) gemv_f32_kernel(const float* __restrict__ A, int lda,
                                                                 const float* __restrict__ W, int N, int K, int M,
                                                                 const int* __restrict__ M_dev, Epi epi) {
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x * GF_WARPS + warp;
  const int nn = n < N ? n : N - 1;
  float4 w[KI];
#pragma unroll
  for (int i = 0; i < KI; ++i) w[i] = __ldg(reinterpret_cast<const float4*>(W + (size_t)nn * K) + lane + 32 * i);
  pdl_wait();
  if (M_dev) M = *M_dev;
  const int r0 = blockIdx.y * GF_MAXM;
  M -= r0;
  A += (size_t)r0 * lda;
  float acc[GF_MAXM];
#pragma unroll
  for (int r = 0; r < GF_MAXM; ++r) {
    acc[r] = 0.f;
    if (r < M) {
      const float4* a = reinterpret_cast<const float4*>(A + (size_t)r * lda);
#pragma unroll
      for (int i = 0; i < KI; ++i) {
        const float4 v = a[lane + 32 * i];
        acc[r] = fmaf(w[i].x, v.x, acc[r]);
        acc[r] = fmaf(w[i].y, v.y, acc[r]);
        acc[r] = fmaf(w[i].z, v.z, acc[r]);
        acc[r] = fmaf(w[i].w, v.w, acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < GF_MAXM; ++r) acc[r] = warp_sum(acc[r]);
  if (lane == 0 && n < N) {
#pragma unroll
    for (int r = 0; r < GF_MAXM; ++r)
      if (r < M) epi.apply1(r0 + r, n, acc[r]);
  }
}

}  // namespace hrt
