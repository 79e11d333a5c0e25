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
