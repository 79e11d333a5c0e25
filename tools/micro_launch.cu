// Cost of a chain of kernels in a CUDA graph, with / without PDL, empty vs. one dependent global load.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__global__ void k_dep(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] = p[blockIdx.x] + 1;
}
int main() {
  int* p;
  cudaMalloc(&p, 1 << 20);
  cudaMemset(p, 0, 1 << 20);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int kind = 0; kind < 2; ++kind)
    for (int pdl = 0; pdl < 2; ++pdl)
      for (int blocks : {1, 148}) {
        const int N = 200;
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = blocks;
          cfg.blockDim = 128;
          cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl;
          cudaLaunchKernelEx(&cfg, kind ? k_dep : k_empty, p);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphExec_t ge;
        cudaGraphInstantiate(&ge, g, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a, st);
          cudaGraphLaunch(ge, st);
          cudaEventRecord(b, st);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
        }
        printf("%s pdl=%d blocks=%3d: %.2f us/kernel\n", kind ? "dep-load" : "empty   ", pdl, blocks, 1000 * ms / N);
      }
  return 0;
}
