// Residual-epilogue write strategies for the fp32 residual stream x[M, 512] (L2-resident, as in
// the encoder): each warp of 148 x 8 warps walks 32 x 32 fp32 chunks like the tcgen05 epilogue.
//   0 rmw     : load x one chunk ahead, add, store (the current EpiResidual)
//   1 red     : red.global.add.v4.f32 (L2 does the read-modify-write)
//   2 tma_red : stage the chunk in smem, cp.reduce.async.bulk.tensor add (TMA reduce)
//   3 store   : plain st.global (write-only bound)
//   4 tma_st  : TMA tile store (write-only bound, async)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_red tools/micro_red.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int D = 512;
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) kern(int mode, float* x, int M, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) float stg_raw[];
  auto stg = reinterpret_cast<float(*)[2][32 * 32]>(stg_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane >> 3, lc = lane & 7;
  const int nchunk = (M / 32) * (D / 32);
  const int gw = blockIdx.x * 8 + warp, nw = gridDim.x * 8;
  float4 pre[8];
  auto addr = [&](int c, int i) {
    const int rb = c / (D / 32), cb = c % (D / 32);
    return x + (size_t)(rb * 32 + lg + 4 * i) * D + cb * 32 + lc * 4;
  };
  if (mode == 0 && gw < nchunk)
#pragma unroll
    for (int i = 0; i < 8; ++i) pre[i] = *reinterpret_cast<const float4*>(addr(gw, i));
  int it = 0;
  for (int c = gw; c < nchunk; c += nw, ++it) {
    const float v = 1.0f;
    if (mode == 0) {
      float4 nx[8];
      const bool more = c + nw < nchunk;
      if (more)
#pragma unroll
        for (int i = 0; i < 8; ++i) nx[i] = *reinterpret_cast<const float4*>(addr(c + nw, i));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 a = pre[i];
        a.x += v; a.y += v; a.z += v; a.w += v;
        *reinterpret_cast<float4*>(addr(c, i)) = a;
      }
      if (more)
#pragma unroll
        for (int i = 0; i < 8; ++i) pre[i] = nx[i];
    } else if (mode == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr(c, i)), "f"(v), "f"(v), "f"(v),
                     "f"(v)
                     : "memory");
    } else if (mode == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<float4*>(addr(c, i)) = make_float4(v, v, v, v);
    } else {
      float* s = stg[warp][it & 1];
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(s + (lg + 4 * i) * 32 + lc * 4) = make_float4(v, v, v, v);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const int rb = c / (D / 32), cb = c % (D / 32);
        if (mode == 2)
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&tm)),
              "r"(su32(s)), "r"(cb * 32), "r"(rb * 32)
              : "memory");
        else
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&tm)),
                       "r"(su32(s)), "r"(cb * 32), "r"(rb * 32)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int M = 29696;
  float* x;
  cudaMalloc(&x, (size_t)M * D * 4);
  cudaMemset(x, 0, (size_t)M * D * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {D, (cuuint64_t)M};
  cuuint64_t strides[1] = {D * 4};
  cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
  CUresult r = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
      &tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tmap failed %d\n", (int)r); return 1; }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[5] = {"rmw", "red", "tma_red", "store", "tma_st"};
  const double mb = (double)M * D * 4 / 1e6;
  for (int grid : {148, 296}) {
    for (int mode = 0; mode < 5; ++mode) {
      cudaMemset(x, 0, (size_t)M * D * 4);
      for (int w = 0; w < 3; ++w) kern<<<grid, 256, 65536>>>(mode, x, M, tm);
      const int reps = 20;
      cudaEventRecord(a);
      for (int i = 0; i < reps; ++i) kern<<<grid, 256, 65536>>>(mode, x, M, tm);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<float> h(4096);
      cudaMemcpy(h.data(), x + (size_t)(M / 2) * D, 4096 * 4, cudaMemcpyDeviceToHost);
      const float expect = (mode == 0 || mode == 1 || mode == 2) ? 23.f : 1.f;
      int bad = 0;
      for (float f : h) bad += f != expect;
      const double us = 1000.0 * ms / reps;
      printf("grid %3d %-8s %7.2f us  %6.0f GB/s of x  (%s)\n", grid, names[mode], us, mb / us * 1e3,
             bad ? "WRONG" : "ok");
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
