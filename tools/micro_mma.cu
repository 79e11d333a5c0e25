// mma.sync m16n8k16 bf16 latency / throughput on sm_100a (one warp, dependent chains)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mg_mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
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
  // 16 warps on one SM, 4 chains each: per-SM throughput
  k<4><<<1, 512>>>(o, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("16 warps x 4 chains: %.2f cycles per mma per SM\n", (double)h / n / 4 / 16);
  return 0;
}
