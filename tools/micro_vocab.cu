// Batch-1 vocabulary GEMV (gemv_vocab_kernel) in isolation: back-to-back
// launches, E L2-resident, R = 1 / 8 rows, V = 32000, K = 512.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2212_01543_b200/csrc tools/micro_vocab.cu -o tools/micro_vocab
#include <cstdio>
#include "gemv_small.cuh"
using namespace hrt;

// pure streaming of each CTA's contiguous E slice (rows * 1 KB), NL loads in flight per thread
template <int NL>
__global__ void __launch_bounds__(512) stream_kernel(const uint4* __restrict__ E, size_t n16_per_cta, float* out) {
  const uint4* base = E + (size_t)blockIdx.x * n16_per_cta;
  uint32_t acc = 0;
  for (size_t i0 = threadIdx.x; i0 < n16_per_cta; i0 += (size_t)blockDim.x * NL) {
    uint4 v[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const size_t i = i0 + (size_t)j * blockDim.x;
      v[j] = i < n16_per_cta ? __ldg(base + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
  }
  if (acc == 0x12345678u) out[blockIdx.x] = 1.f;
}

// gemv_vocab's load pattern without the MMAs / statistics (NB chunks in flight per batch)
template <int NB>
__global__ void __launch_bounds__(512) pattern_kernel(const bf16* __restrict__ E, int V, int K, float* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int n0 = blockIdx.x * GV_VTILE + warp * 16;
  const int nch = K / 32;
  const bf16* w0 = E + (size_t)max(0, min(n0 + g, V - 1)) * K + t4 * 8;
  const bf16* w1 = E + (size_t)max(0, min(n0 + g + 8, V - 1)) * K + t4 * 8;
  const uint64_t pol = gv_policy();
  uint32_t acc = 0;
  for (int cb = 0; cb < nch; cb += NB) {
    uint4 u0[NB], u1[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int ch = min(cb + i, nch - 1);
      u0[i] = gv_ldw(w0 + 32 * ch, pol);
      u1[i] = gv_ldw(w1 + 32 * ch, pol);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) acc ^= u0[i].x ^ u1[i].y ^ u0[i].z ^ u1[i].w;
  }
  if (acc == 0x12345678u) out[blockIdx.x] = 1.f;
}

// fragment-native layout: a warp's 16 rows x K stored so that load (chunk, half) of all
// 32 lanes is one contiguous 512-byte run
template <int NB>
__global__ void __launch_bounds__(512) native_kernel(const bf16* __restrict__ E, int V, int K, float* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * GV_VTILE + warp * 16;
  const int nch = K / 32;
  const bf16* wb = E + (size_t)min(n0, V - 16) * K;  // 16 rows x K, fragment-ordered
  const uint64_t pol = gv_policy();
  uint32_t acc = 0;
  for (int cb = 0; cb < nch; cb += NB) {
    uint4 u0[NB], u1[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int ch = min(cb + i, nch - 1);
      u0[i] = gv_ldw(wb + ((size_t)(2 * ch) * 32 + lane) * 8, pol);
      u1[i] = gv_ldw(wb + ((size_t)(2 * ch + 1) * 32 + lane) * 8, pol);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) acc ^= u0[i].x ^ u1[i].y ^ u0[i].z ^ u1[i].w;
  }
  if (acc == 0x12345678u) out[blockIdx.x] = 1.f;
}

int main() {
  const int V = 32000, K = 512;
  bf16 *E, *A;
  cudaMalloc(&E, (size_t)V * K * 2);
  cudaMalloc(&A, (size_t)64 * K * 2);
  cudaMemset(E, 0x11, (size_t)V * K * 2);
  cudaMemset(A, 0x22, (size_t)64 * K * 2);
  const int nt = (V + GV_VTILE - 1) / GV_VTILE;
  VocabParts p;
  cudaMalloc(&p.mx, 64 * nt * 4);
  cudaMalloc(&p.sum, 64 * nt * 4);
  cudaMalloc(&p.val, 64 * nt * 4);
  cudaMalloc(&p.id, 64 * nt * 4);
  cudaMalloc(&p.eos, 64 * 4);
  p.ntiles = nt;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int M : {1, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      for (int w = 0; w < 5; ++w)
        gemv_vocab_kernel<1, false><<<nt, GV_VWARPS * 32>>>(A, K, E, V, K, M, nullptr, p, 0, GvLN{nullptr, nullptr, nullptr});
      cudaEventRecord(a);
      const int it = 200;
      for (int w = 0; w < it; ++w)
        gemv_vocab_kernel<1, false><<<nt, GV_VWARPS * 32>>>(A, K, E, V, K, M, nullptr, p, 0, GvLN{nullptr, nullptr, nullptr});
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("gemv_vocab M=%d: %.2f us/launch (%.0f GB/s of E)\n", M, 1000 * ms / it, (double)V * K * 2 / (ms / it * 1e-3) / 1e9);
    }
  }
  for (int ctas : {125, 148, 250, 296}) {
    const size_t per = ((size_t)V * K * 2 / 16 + ctas - 1) / ctas;
    float* o;
    cudaMalloc(&o, 4096);
    for (int w = 0; w < 5; ++w) stream_kernel<16><<<ctas, 512>>>(reinterpret_cast<const uint4*>(E), per, o);
    cudaEventRecord(a);
    for (int w = 0; w < 200; ++w) stream_kernel<16><<<ctas, 512>>>(reinterpret_cast<const uint4*>(E), per, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("stream %d CTAs x 512 thr, 16 loads in flight: %.2f us/launch (%.0f GB/s)\n", ctas, 1000 * ms / 200,
           (double)V * K * 2 / (ms / 200 * 1e-3) / 1e9);
  }
  for (int nb : {8, 16}) {
    float* o;
    cudaMalloc(&o, 4096);
    auto go = [&]() {
      if (nb == 8) pattern_kernel<8><<<nt, GV_VWARPS * 32>>>(E, V, K, o);
      else pattern_kernel<16><<<nt, GV_VWARPS * 32>>>(E, V, K, o);
    };
    for (int w = 0; w < 5; ++w) go();
    cudaEventRecord(a);
    for (int w = 0; w < 200; ++w) go();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("gemv load pattern only, %d chunks per batch: %.2f us/launch\n", nb, 1000 * ms / 200);
  }
  for (int nb : {8, 16}) {
    float* o;
    cudaMalloc(&o, 4096);
    auto go = [&]() {
      if (nb == 8) native_kernel<8><<<nt, GV_VWARPS * 32>>>(E, V, K, o);
      else native_kernel<16><<<nt, GV_VWARPS * 32>>>(E, V, K, o);
    };
    for (int w = 0; w < 5; ++w) go();
    cudaEventRecord(a);
    for (int w = 0; w < 200; ++w) go();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("fragment-native layout, %d chunks per batch: %.2f us/launch\n", nb, 1000 * ms / 200);
  }
  // empty-kernel launch floor
  {
    float* o;
    cudaMalloc(&o, 4096);
    for (int w = 0; w < 5; ++w) stream_kernel<1><<<148, 512>>>(reinterpret_cast<const uint4*>(E), 0, o);
    cudaEventRecord(a);
    for (int w = 0; w < 200; ++w) stream_kernel<1><<<148, 512>>>(reinterpret_cast<const uint4*>(E), 0, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel 148x512: %.2f us/launch\n", 1000 * ms / 200);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
