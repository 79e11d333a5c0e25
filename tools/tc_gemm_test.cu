// Standalone check of the tcgen05 GEMM (tc_gemm.cuh) against a CPU fp64 dot
// product on sampled entries, plus a timing line per shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2212_01543_b200/csrc \
//        tools/tc_gemm_test.cu -o tools/tc_gemm_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <type_traits>
#include "tc_gemm.cuh"
#include "kernels.cuh"
#include "tmap.h"

using namespace hrt;

struct StoreEpi {
  static constexpr bool kRowWise = false;
  float* C;
  int ldc;
  __device__ void apply8(int row0, int col, const float4* v, int M) const {
    for (int i = 0; i < 8; ++i)
      if (row0 + 4 * i < M) *reinterpret_cast<float4*>(C + (size_t)(row0 + 4 * i) * ldc + col) = v[i];
  }
};

// timing-only epilogue: drops the accumulator (isolates the TMA + MMA mainloop)
struct NullEpi {
  static constexpr bool kRowWise = false;
  float* C;
  int ldc;
  __device__ void apply8(int row0, int col, const float4* v, int M) const {
    if (v[0].x == 123456.f && row0 < 0) C[col] = v[1].y;
  }
};

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int BN, int ST, int CL = 1, class E = StoreEpi>
bool run(int M, int N, int K) {
  std::mt19937 g(M * 7 + N * 3 + K);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<__nv_bfloat16> hA((size_t)M * K), hB((size_t)N * K);
  for (auto& x : hA) x = __float2bfloat16(nd(g));
  for (auto& x : hB) x = __float2bfloat16(nd(g));
  __nv_bfloat16 *dA, *dB;
  float* dC;
  CK(cudaMalloc(&dA, hA.size() * 2));
  CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0xff, (size_t)M * N * 4));
  CUtensorMap ta = make_tmap_bf16_kmajor(dA, M, K, K, TC_BM);
  CUtensorMap tb = make_tmap_bf16_kmajor(dB, N, K, K, BN / CL);
  auto kern = tc_gemm_kernel<BN, ST, E, CL>;
  int smem = TcSmem<BN, ST>::TOTAL;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int tiles = ((N + BN - 1) / BN) * ((M + TC_BM * CL - 1) / (TC_BM * CL)) * CL;
  dim3 grid(tiles < nsm / CL * CL ? tiles : nsm / CL * CL);
  E epi{dC, N};
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
  auto go = [&]() { CK(cudaLaunchKernelEx(&cfg, kern, ta, tb, ta, M, N, K, (const int*)nullptr, epi, SplitK{1, nullptr, nullptr})); };
  go();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> hC((size_t)M * N);
  CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  int bad = 0;
  std::uniform_int_distribution<int> um(0, M - 1), un(0, N - 1);
  for (int s = 0; s < 4000; ++s) {
    int i = s < 64 ? (s % M) : um(g), j = s < 64 ? ((s * 37) % N) : un(g);
    double ref = 0;
    for (int k = 0; k < K; ++k)
      ref += (double)__bfloat162float(hA[(size_t)i * K + k]) * (double)__bfloat162float(hB[(size_t)j * K + k]);
    double err = fabs(ref - hC[(size_t)i * N + j]) / (1.0 + fabs(ref));
    if (err > maxerr) maxerr = err;
    if (err > 1e-3 && !std::is_same<E, NullEpi>::value) {
      if (bad < 5) printf("   mismatch C[%d,%d] = %f ref %f\n", i, j, hC[(size_t)i * N + j], ref);
      ++bad;
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) go();
  cudaEventRecord(e0);
  const int iters = 20;
  for (int w = 0; w < iters; ++w) go();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double us = ms * 1000.0 / iters;
  double tflops = 2.0 * M * N * K / (us * 1e-6) / 1e12;
  double gbs = ((double)M * K * 2 + (double)N * K * 2 + (double)M * N * 4) / (us * 1e-6) / 1e9;
  printf("%s CL=%d BN=%3d ST=%d M=%6d N=%6d K=%5d : maxrel=%.2e bad=%d  %.2f us  %.1f TFLOP/s  %.0f GB/s  %s\n", std::is_same<E, NullEpi>::value ? "null " : "store", CL, BN, ST, M,
         N, K, maxerr, bad, us, tflops, gbs, bad ? "FAIL" : "ok");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return bad == 0;
}

// timing of the fused vocabulary epilogue (row-wise softmax statistics + top-1)
template <int CL>
void time_vocab(int M, int N, int K) {
  __nv_bfloat16 *dA, *dB;
  CK(cudaMalloc(&dA, (size_t)M * K * 2));
  CK(cudaMalloc(&dB, (size_t)N * K * 2));
  CK(cudaMemset(dA, 0x11, (size_t)M * K * 2));
  CK(cudaMemset(dB, 0x22, (size_t)N * K * 2));
  const int bn = 128, nt = (N + bn - 1) / bn;
  VocabParts parts;
  CK(cudaMalloc(&parts.mx, (size_t)M * nt * 4));
  CK(cudaMalloc(&parts.sum, (size_t)M * nt * 4));
  CK(cudaMalloc(&parts.val, (size_t)M * nt * 4));
  CK(cudaMalloc(&parts.id, (size_t)M * nt * 4));
  CK(cudaMalloc(&parts.eos, (size_t)M * 4));
  parts.ntiles = nt;
  VocabEpi<1> epi{parts, 0, bn};
  CUtensorMap ta = make_tmap_bf16_kmajor(dA, M, K, K, TC_BM);
  CUtensorMap tb = make_tmap_bf16_kmajor(dB, N, K, K, 256 / CL);
  auto kern = tc_gemm_kernel<256, 4, VocabEpi<1>, CL>;
  int smem = TcSmem<256, 4>::TOTAL;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int tiles = ((N + 255) / 256) * ((M + TC_BM * CL - 1) / (TC_BM * CL)) * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles < 148 / CL * CL ? tiles : 148 / CL * CL);
  cfg.blockDim = TC_THREADS;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&]() { CK(cudaLaunchKernelEx(&cfg, kern, ta, tb, ta, M, N, K, (const int*)nullptr, epi, SplitK{1, nullptr, nullptr})); };
  for (int w = 0; w < 3; ++w) go();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int w = 0; w < 20; ++w) go();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1000.0 / 20;
  printf("vocab CL=%d M=%6d N=%6d K=%5d : %.2f us  %.1f TFLOP/s\n", CL, M, N, K, us, 2.0 * M * N * K / (us * 1e-6) / 1e12);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(parts.mx);
  cudaFree(parts.sum);
  cudaFree(parts.val);
  cudaFree(parts.id);
  cudaFree(parts.eos);
}

int main() {
  time_vocab<1>(1024, 32000, 512);
  time_vocab<2>(1024, 32000, 512);
  time_vocab<1>(512, 32000, 512);
  time_vocab<2>(22528, 32000, 512);
  bool ok = true;
  ok &= run<32, 8>(1, 256, 64);
  ok &= run<32, 8>(800, 384, 128);
  ok &= run<32, 8>(1000, 512, 512);
  ok &= run<32, 8>(100, 64, 128);
  ok &= run<64, 8>(800, 384, 128);
  ok &= run<256, 4>(1, 256, 64);
  ok &= run<128, 6>(1000, 640, 512);
  ok &= run<256, 4>(1, 32000, 512);
  ok &= run<256, 4>(200, 512, 512);
  ok &= run<256, 4>(1000, 1536, 512);
  ok &= run<128, 6>(300, 2048, 512);
  ok &= run<64, 8>(64, 512, 2048);
  ok &= run<128, 6>(30000, 512, 512);
  ok &= run<128, 6>(30000, 1536, 512);
  ok &= run<128, 6>(30000, 2048, 512);
  ok &= run<128, 6>(30000, 512, 2048);
  ok &= run<256, 4>(1024, 32000, 512);
  ok &= run<256, 4>(8192, 2048, 512);
  ok &= run<256, 4>(8192, 512, 2048);
  ok &= run<128, 6>(8192, 512, 2048);
  // CTA pairs with multicast B halves
  ok &= run<256, 4, 2>(1, 256, 64);
  ok &= run<256, 4, 2>(200, 512, 512);
  ok &= run<256, 4, 2>(1000, 1536, 512);
  ok &= run<64, 8, 2>(800, 384, 128);
  ok &= run<32, 8, 2>(1000, 512, 512);
  ok &= run<128, 6, 2>(1000, 640, 512);
  ok &= run<256, 4, 2>(1024, 32000, 512);
  ok &= run<256, 4>(29300, 1536, 512);
  ok &= run<256, 4, 2>(29300, 1536, 512);
  ok &= run<256, 4>(29300, 512, 512);
  ok &= run<256, 4, 2>(29300, 512, 512);
  ok &= run<256, 4>(29300, 2048, 512);
  ok &= run<256, 4, 2>(29300, 2048, 512);
  ok &= run<256, 4>(29300, 512, 2048);
  ok &= run<256, 4, 2>(29300, 512, 2048);
  ok &= run<128, 6, 2>(29300, 512, 2048);
  ok &= run<256, 4, 1, NullEpi>(1024, 32000, 512);
  ok &= run<256, 4, 2, NullEpi>(1024, 32000, 512);
  ok &= run<256, 4, 1, NullEpi>(512, 32000, 512);
  ok &= run<256, 4, 2, NullEpi>(512, 32000, 512);
  ok &= run<256, 4, 1, NullEpi>(29300, 512, 2048);
  ok &= run<256, 4, 2, NullEpi>(29300, 512, 2048);
  ok &= run<256, 4, 1, NullEpi>(29300, 2048, 512);
  ok &= run<256, 4, 2, NullEpi>(29300, 2048, 512);
  ok &= run<256, 4, 1, NullEpi>(29600, 2048, 2048);
  ok &= run<256, 4, 2, NullEpi>(29600, 2048, 2048);
  ok &= run<256, 4, 2, NullEpi>(37888, 2048, 2048);
  printf(ok ? "ALL OK\n" : "SOME FAILED\n");
  return ok ? 0 : 1;
}
