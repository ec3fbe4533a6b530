// mma.sync.m8n8k4 f64 (DMMA) on sm_100a: fragment-layout check against the host, and the
// issue cost of a chain. Layout assumed: A (8x4, row): lane -> (lane>>2, lane&3);
// B (4x8, col): lane -> (k = lane&3, n = lane>>2); C/D (8x8): lane -> (lane>>2, 2*(lane&3)+{0,1}).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__global__ void k_check(const double *A, const double *B, double *C) {
  const int lane = threadIdx.x;
  const double a = A[(lane >> 2) * 4 + (lane & 3)];     // A row-major 8x4
  const double b = B[(lane & 3) * 8 + (lane >> 2)];     // B row-major 4x8: (k, n)
  double d0, d1;
  dmma(d0, d1, a, b, 0.0, 0.0);
  C[(lane >> 2) * 8 + 2 * (lane & 3)] = d0;
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
}
__global__ void k_time(double *out, int reps, long long *cyc) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 0.5, c[6] = {0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int t = 0; t < 3; ++t) dmma(c[2 * t], c[2 * t + 1], a, b, c[2 * t], c[2 * t + 1]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3] + c[4] + c[5];
}
int main() {
  double hA[32], hB[32], hC[64], *dA, *dB, *dC;
  for (int i = 0; i < 32; ++i) { hA[i] = 0.1 * i - 1.3; hB[i] = 0.07 * i * i - 0.5; }
  cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  k_check<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double r = 0; for (int k = 0; k < 4; ++k) r += hA[i * 4 + k] * hB[k * 8 + j];
      err = fmax(err, fabs(r - hC[i * 8 + j]));
    }
  printf("layout check max err %.3e (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
  double *o; long long *cy; cudaMalloc(&o, 1 << 20); cudaMallocManaged(&cy, 8 * 1024);
  for (int warps : {1, 4, 16}) {
    k_time<<<1, 32 * warps>>>(o, 1000, cy); cudaDeviceSynchronize();
    k_time<<<1, 32 * warps>>>(o, 1000, cy); cudaDeviceSynchronize();
    printf("warps %2d: %lld cycles per 3 independent DMMA chains step (per warp)\n", warps, cy[0]);
  }
  return 0;
}
