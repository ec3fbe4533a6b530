// Per-node cost of dependent kernel launches inside a CUDA graph vs grid-wide barriers
// inside one persistent cooperative kernel (148 CTAs x 256 threads, B200).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_small(double *x, int n) {   // one light pass over n doubles
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = x[i] * 0.999 + 1.0;
}
__global__ void k_coop(double *x, int n, int reps) {
  cg::grid_group g = cg::this_grid();
  for (int r = 0; r < reps; ++r) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = x[i] * 0.999 + 1.0;
    g.sync();
  }
}
int main() {
  const int n = 50000, reps = 200;
  double *x; cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {148, 296, 592}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int r = 0; r < reps; ++r) k_small<<<grid, 256, 0, s>>>(x, n);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s); for (int t = 0; t < 5; ++t) cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of dependent kernels, grid %d: %.2f us per kernel\n", grid, ms * 1000 / (5 * reps));
  }
  for (int grid : {148, 296}) {
    void *args[] = {&x, (void *)&n, (void *)&reps};
    cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    for (int t = 0; t < 5; ++t) cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cooperative kernel, grid %d: %.2f us per pass + grid.sync (%s)\n", grid, ms * 1000 / (5 * reps), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
