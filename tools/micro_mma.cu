// mma.sync m16n8k16 bf16 latency / throughput on sm_100a (one warp, dependent chains)
#include <cstdio>
#include "../paper_2212_01543_b200/csrc/decode_mega.cuh"
using namespace hrt;
template <int CH>
__global__ void k(float* out, int n, long long* cyc) {
  float c[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) mg_mma(c[j], a0, a1, a2, a3, b0, b1);
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  long long h;
  const int n = 1000;
  k<1><<<1, 32>>>(o, n, c); cudaDeviceSynchronize();
  k<1><<<1, 32>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("1 chain: %.1f cycles/mma\n", (double)h / n);
  k<2><<<1, 32>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("2 chains: %.1f cycles/mma\n", (double)h / n / 2);
  k<4><<<1, 32>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("4 chains: %.1f cycles/mma\n", (double)h / n / 4);
  k<8><<<1, 32>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("8 chains: %.1f cycles/mma\n", (double)h / n / 8);
  return 0;
}
