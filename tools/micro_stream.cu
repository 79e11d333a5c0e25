// Per-SM weight-streaming rate from L2 (the decode-cluster kernel's limit):
// G CTAs (one per SM) each stream BYTES of a buffer (L2-warm after the first
// rep) into shared memory and touch every 16 bytes, under three mechanisms:
//   0 bulk  : cp.async.bulk 1-D copies into an NSLOT x CHUNK ring (mbarrier complete_tx)
//   1 ldgsts: cp.async.cg 16 B per thread into the same ring (commit groups)
//   2 ldg   : ld.global.v4 straight into registers, UNROLL loads in flight per thread
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_stream tools/micro_stream.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(n), "r"(su32(bar))
               : "memory");
}

template <int MODE, int CHUNK, int NSLOT>
__global__ void __launch_bounds__(256) kern(const uint4* __restrict__ src, size_t per_cta, float* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[NSLOT];
  const uint8_t* base = reinterpret_cast<const uint8_t*>(src) + per_cta * blockIdx.x;
  const int nch = (int)(per_cta / CHUNK);
  float acc = 0.f;
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < NSLOT; ++s) mbar_init(&full[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < NSLOT && i < nch; ++i) {
        mbar_expect(&full[i], CHUNK);
        bulk(ring + i * CHUNK, base + (size_t)i * CHUNK, CHUNK, &full[i]);
      }
    for (int i = 0; i < nch; ++i) {
      const int s = i % NSLOT;
      mbar_wait(&full[s], (i / NSLOT) & 1);
      const uint4* r = reinterpret_cast<const uint4*>(ring + s * CHUNK);
      for (int j = threadIdx.x; j < CHUNK / 16; j += 256) acc += __uint_as_float(r[j].x);
      __syncthreads();
      if (threadIdx.x == 0 && i + NSLOT < nch) {
        mbar_expect(&full[s], CHUNK);
        bulk(ring + s * CHUNK, base + (size_t)(i + NSLOT) * CHUNK, CHUNK, &full[s]);
      }
    }
  } else if (MODE == 1) {
    auto issue = [&](int i) {
      const int s = i % NSLOT;
      for (int j = threadIdx.x; j < CHUNK / 16; j += 256)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(ring + s * CHUNK + 16 * j)),
                     "l"(base + (size_t)i * CHUNK + 16 * j)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < NSLOT - 1 && i < nch; ++i) issue(i);
    for (int i = 0; i < nch; ++i) {
      if (i + NSLOT - 1 < nch) issue(i + NSLOT - 1);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(NSLOT - 1) : "memory");
      __syncthreads();
      const uint4* r = reinterpret_cast<const uint4*>(ring + (i % NSLOT) * CHUNK);
      for (int j = threadIdx.x; j < CHUNK / 16; j += 256) acc += __uint_as_float(r[j].x);
      __syncthreads();
    }
  } else {
    constexpr int U = NSLOT;  // loads in flight per thread
    const uint4* p = reinterpret_cast<const uint4*>(base);
    const int n16 = (int)(per_cta / 16);
    for (int j0 = threadIdx.x; j0 < n16; j0 += 256 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = j0 + 256 * u < n16 ? __ldcg(p + j0 + 256 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x);
    }
  }
  if (acc == 12345.f) sink[blockIdx.x] = acc;
}

template <int MODE, int CHUNK, int NSLOT>
void run(const char* name, const uint4* buf, float* sink, int G, size_t per_cta) {
  auto k = kern<MODE, CHUNK, NSLOT>;
  const int smem = MODE == 2 ? 0 : CHUNK * NSLOT;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k<<<G, 256, smem>>>(buf, per_cta, sink);
  const int reps = 50;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) k<<<G, 256, smem>>>(buf, per_cta, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1000.0 * ms / reps;
  printf("%-22s G=%3d %4zu KB/CTA: %7.2f us/launch  %6.1f GB/s per SM  %7.1f GB/s total  (%s)\n", name, G,
         per_cta / 1024, us, per_cta / us / 1e3, per_cta * G / us / 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint4* buf;
  float* sink;
  const size_t total = 64ull << 20;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 0, total);
  cudaMalloc(&sink, 4096);
  // per-CTA volume large enough to amortise the launch (all of it L2-resident: <= 56 MB)
  for (int G : {1, 16, 32, 148}) {
    const size_t per = (size_t)(G == 148 ? 384 : (G == 32 ? 1792 : 3584)) << 10;
    run<0, 32768, 5>("bulk 5x32KB", buf, sink, G, per);
    run<0, 16384, 10>("bulk 10x16KB", buf, sink, G, per);
    run<1, 16384, 8>("ldgsts 8x16KB", buf, sink, G, per);
    run<2, 16, 8>("ldg 8/thread", buf, sink, G, per);
    run<2, 16, 16>("ldg 16/thread", buf, sink, G, per);
  }
  return 0;
}
