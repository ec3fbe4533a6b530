// Per-kernel cost of a chain of dependent kernel launches inside a CUDA graph (B200):
// empty kernels of G CTAs x 256 threads, and the same with programmatic dependent launch.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int *p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1; }
__global__ void k_empty_pdl(int *p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
int main() {
  int *d; cudaMalloc(&d, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int G : {1, 148, 592, 2048}) {
      const int K = 40;
      cudaGraph_t g; cudaGraphExec_t e;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < K; ++k) {
        if (!pdl) k_empty<<<G, 256, 0, s>>>(d);
        else {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = G; cfg.blockDim = 256; cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, k_empty_pdl, d);
        }
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&e, g, 0);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(e, s);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int r = 0; r < 50; ++r) cudaGraphLaunch(e, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("pdl %d grid %5d: %.2f us per dependent kernel (%s)\n", pdl, G, ms * 1000 / (50.0 * K),
             cudaGetErrorString(cudaGetLastError()));
      cudaGraphExecDestroy(e); cudaGraphDestroy(g);
    }
  return 0;
}
