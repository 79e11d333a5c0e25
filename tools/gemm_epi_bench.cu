// tcgen05 GEMM: mainloop vs epilogue cost at the encoder shapes (B = 1024: M ~ 30k).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2212_01543_b200/csrc tools/gemm_epi_bench.cu -o tools/gemm_epi_bench -lcuda
#include <cstdio>
#include <vector>
#include "tc_gemm.cuh"
#include "gemm_epi.cuh"
#include "tmap.h"
using namespace hrt;

struct NullEpi {
  static constexpr bool kRowWise = false;
  float* sink;
  __device__ void apply8(int row0, int col, const float4* v, int M) const {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += v[i].x;
    if (s == 1234.5f) sink[0] = s;  // keep the TMEM loads alive, no stores
  }
};

// row-store variants (lane = row, 32 consecutive columns)
struct RowBias {
  static constexpr bool kRowWise = false;
  static constexpr bool kRowStore = true;
  bf16* out;
  int ldo;
  const float* bias;
  __device__ void apply8(int, int, const float4*, int) const {}
  __device__ __forceinline__ void row32(int row, int col0, const float* v, int nvalid) const {
    bf16* o = out + (size_t)row * ldo + col0;
    if (nvalid >= 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col0 + q * 8 + (e & 2) * 2));
          const float bx = (e & 1) ? b.z : b.x, by = (e & 1) ? b.w : b.y;
          __nv_bfloat162 h = __floats2bfloat162_rn(v[q * 8 + 2 * e] + bx, v[q * 8 + 2 * e + 1] + by);
          w[e] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(o + q * 8) = u;
      }
    }
  }
};
struct RowResidual {
  static constexpr bool kRowWise = false;
  static constexpr bool kRowStore = true;
  float* x;
  int ldx;
  const float* bias;
  __device__ void apply8(int, int, const float4*, int) const {}
  __device__ __forceinline__ void row32(int row, int col0, const float* v, int nvalid) const {
    float* p = x + (size_t)row * ldx + col0;
    if (nvalid >= 32) {
      float4 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = reinterpret_cast<const float4*>(p)[q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col0) + q);
        a[q].x += v[4 * q] + b.x;
        a[q].y += v[4 * q + 1] + b.y;
        a[q].z += v[4 * q + 2] + b.z;
        a[q].w += v[4 * q + 3] + b.w;
        reinterpret_cast<float4*>(p)[q] = a[q];
      }
    }
  }
};

template <int BN, int ST, class Epi, int CL = 1>
double timeit(int M, int N, int K, const bf16* A, const bf16* B, const Epi& epi) {
  CUtensorMap ta = make_tmap_bf16_kmajor(A, M, K, K, TC_BM);
  CUtensorMap tb = make_tmap_bf16_kmajor(B, N, K, K, BN / CL);
  auto kern = tc_gemm_kernel<BN, ST, Epi, CL>;
  int smem = TcSmem<BN, ST>::TOTAL;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int tiles = ((N + BN - 1) / BN) * ((M + TC_BM * CL - 1) / (TC_BM * CL)) * CL;
  dim3 grid(tiles < 148 ? tiles : 148);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = TC_THREADS;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // output tile map for the TMA-store epilogue (EpiBiasT<bf16>); other epilogues ignore it
  CUtensorMap tc = ta;
  if constexpr (EpiTmaStore<Epi>::value) tc = make_tmap_bf16_store(epi.out, M, N, epi.ldo);
  auto go = [&]() { cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, M, N, K, (const int*)nullptr, epi, SplitK{1, nullptr, nullptr}); };
  for (int w = 0; w < 3; ++w) go();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) go();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.0 / it;
}

int main() {
  const int M = 29696;
  bf16 *A, *B, *C;
  float *x, *bias, *sink;
  cudaMalloc(&A, (size_t)M * 2048 * 2);
  cudaMalloc(&B, (size_t)2048 * 2048 * 2);
  cudaMalloc(&C, (size_t)M * 2048 * 2);
  cudaMalloc(&x, (size_t)M * 512 * 4);
  cudaMalloc(&bias, 2048 * 4);
  cudaMalloc(&sink, 64);
  cudaMemset(A, 0, (size_t)M * 2048 * 2);
  cudaMemset(B, 0, (size_t)2048 * 2048 * 2);
  cudaMemset(bias, 0, 2048 * 4);
  struct S { int N, K; const char* name; } shapes[] = {{1536, 512, "QKV"}, {512, 512, "Wo"}, {2048, 512, "W1"}, {512, 2048, "W2"}};
  for (auto sh : shapes) {
    const double fl = 2.0 * M * sh.N * sh.K;
    NullEpi ne{sink};
    EpiBiasT<bf16, false> eb{C, sh.N, bias};
    EpiResidual er{x, 512, bias};
    double t1 = timeit<256, 4>(M, sh.N, sh.K, A, B, ne);
    double t2 = timeit<128, 6>(M, sh.N, sh.K, A, B, ne);
    double t3, t4;
    if (sh.N == 512) {
      t3 = timeit<256, 4>(M, sh.N, sh.K, A, B, er);
      t4 = timeit<128, 6>(M, sh.N, sh.K, A, B, er);
    } else {
      t3 = timeit<256, 4>(M, sh.N, sh.K, A, B, eb);
      t4 = timeit<128, 6>(M, sh.N, sh.K, A, B, eb);
    }
    double t5, t6, t7;
    if (sh.N == 512) {
      RowResidual rr{x, 512, bias};
      t5 = timeit<256, 4>(M, sh.N, sh.K, A, B, rr);
      t6 = timeit<256, 4, EpiResidual, 2>(M, sh.N, sh.K, A, B, er);
    } else {
      RowBias rb{C, sh.N, bias};
      t5 = timeit<256, 4>(M, sh.N, sh.K, A, B, rb);
      t6 = timeit<256, 4, EpiBiasT<bf16, false>, 2>(M, sh.N, sh.K, A, B, eb);
    }
    t7 = timeit<256, 4, NullEpi, 2>(M, sh.N, sh.K, A, B, ne);
    printf("%-4s M=%d N=%d K=%d | null: BN256 %.1f us (%.0f TF) BN128 %.1f (%.0f) CL2 %.1f (%.0f) | real: BN256 %.1f us (%.0f TF) BN128 %.1f (%.0f) CL2 %.1f (%.0f) | row-store BN256 %.1f (%.0f)\n",
           sh.name, M, sh.N, sh.K, t1, fl / t1 / 1e6, t2, fl / t2 / 1e6, t7, fl / t7 / 1e6, t3, fl / t3 / 1e6, t4, fl / t4 / 1e6, t6, fl / t6 / 1e6, t5, fl / t5 / 1e6);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
