// Microbenchmarks for the persistent decode kernel design: grid-barrier cost
// and GEMV-phase throughput at R = 1 on a 148-CTA persistent grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro_mega tools/micro_mega.cu
#include <cstdio>
#include <vector>

#include "../paper_2212_01543_b200/csrc/decode_mega.cuh"

using namespace hrt;

// monotonic-count barrier: one red.release per CTA, spin with ld.acquire
__device__ __forceinline__ void bar_mono(unsigned* cnt, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
    } while ((int)(cur - target) < 0);
  }
  __syncthreads();
}

// flag barrier: CTA c publishes epoch in its own line; CTA 0 gathers, then broadcasts
__device__ __forceinline__ void bar_flags(unsigned* flags, unsigned* go, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(epoch) : "memory");
  if (blockIdx.x == 0) {
    for (int c = threadIdx.x; c < gridDim.x; c += blockDim.x) {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(flags + c * 32) : "memory");
      } while (cur != epoch);
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(epoch) : "memory");
  } else if (threadIdx.x == 0) {
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(go) : "memory");
    } while (cur != epoch);
  }
  __syncthreads();
}
// two-level counter: groups of 16 CTAs share a counter; group leaders bump the top counter
__device__ __forceinline__ void bar_tree(unsigned* cnt, unsigned round) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int grp = blockIdx.x >> 4, ngrp = (gridDim.x + 15) >> 4;
    const int gsize = min(16, (int)gridDim.x - grp * 16);
    unsigned* gc = cnt + 64 + grp * 32;
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(gc), "r"(1) : "memory");
    if (old == round * gsize + gsize - 1)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt), "r"(1) : "memory");
    unsigned cur;
    const unsigned target = (round + 1) * ngrp;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory");
    } while ((int)(cur - target) < 0);
  }
  __syncthreads();
}
template <int V>
__device__ __forceinline__ void bar_var(unsigned* cnt, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V == 0) {  // relaxed arrive/poll, no fences (latency floor; NOT a valid barrier for data)
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned cur;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory"); } while ((int)(cur - target) < 0);
    } else if (V == 1) {  // fence.acq_rel + relaxed arrive, relaxed poll, fence.acq_rel after
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned cur;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory"); } while ((int)(cur - target) < 0);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    } else {  // release arrive, relaxed poll, acquire fence after
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned cur;
      do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(cnt) : "memory"); } while ((int)(cur - target) < 0);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  __syncthreads();
}
template <int V>
__global__ void __launch_bounds__(MG_THREADS, 1) k_bar_var(unsigned* cnt, int iters) {
  for (int i = 0; i < iters; ++i) bar_var<V>(cnt, (unsigned)(i + 1) * gridDim.x);
}
__global__ void __launch_bounds__(MG_THREADS, 1) k_bar_flags(unsigned* flags, int iters) {
  for (int i = 0; i < iters; ++i) bar_flags(flags, flags + 32 * 200, (unsigned)i + 1);
}
__global__ void __launch_bounds__(MG_THREADS, 1) k_bar_tree(unsigned* cnt, int iters) {
  for (int i = 0; i < iters; ++i) bar_tree(cnt, (unsigned)i);
}
__global__ void __launch_bounds__(MG_THREADS, 1) k_bar_old(unsigned* bar, int iters) {
  unsigned target = 0;
  for (int i = 0; i < iters; ++i) mg_sync(bar, target);
}
__global__ void __launch_bounds__(MG_THREADS, 1) k_bar_mono(unsigned* cnt, int iters) {
  for (int i = 0; i < iters; ++i) bar_mono(cnt, (unsigned)(i + 1) * gridDim.x);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  cudaMalloc(&bar, 64);
  unsigned* flags;
  cudaMalloc(&flags, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int it = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(bar, 0, 64);
    cudaEventRecord(a);
    k_bar_old<<<sms, MG_THREADS>>>(bar, it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mg_sync barrier: %.3f us/barrier\n", 1000 * ms / it);
    cudaMemset(bar, 0, 64);
    cudaEventRecord(a);
    k_bar_mono<<<sms, MG_THREADS>>>(bar, it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mono barrier: %.3f us/barrier\n", 1000 * ms / it);
    cudaMemset(flags, 0, 1 << 20);
    cudaEventRecord(a);
    k_bar_flags<<<sms, MG_THREADS>>>(flags, it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("flag barrier: %.3f us/barrier\n", 1000 * ms / it);
    cudaMemset(flags, 0, 1 << 20);
    cudaEventRecord(a);
    k_bar_tree<<<sms, MG_THREADS>>>(flags, it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("tree barrier: %.3f us/barrier\n", 1000 * ms / it);
    for (int v = 0; v < 3; ++v) {
      cudaMemset(bar, 0, 64);
      cudaEventRecord(a);
      if (v == 0) k_bar_var<0><<<sms, MG_THREADS>>>(bar, it);
      if (v == 1) k_bar_var<1><<<sms, MG_THREADS>>>(bar, it);
      if (v == 2) k_bar_var<2><<<sms, MG_THREADS>>>(bar, it);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("variant %d barrier: %.3f us/barrier\n", v, 1000 * ms / it);
    }
    for (int nb : {74, 37}) {
      cudaMemset(bar, 0, 64);
      cudaEventRecord(a);
      k_bar_mono<<<nb, MG_THREADS>>>(bar, it);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("mono barrier %d CTAs: %.3f us/barrier\n", nb, 1000 * ms / it);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
