// Latency microbenchmarks (dependent chains, one warp) for the K-EIG design.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double *out, long long *cyc, double seed) {
  __shared__ double sm[64];
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  float f = (float)seed;
  sm[threadIdx.x] = x;
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // shfl double chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffff, x, 1);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // LDS.64 dependent chain (pointer chase via index from value)
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { double v = sm[idx]; idx = ((int)v & 31) ^ (threadIdx.x & 31); x += v; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // F2F double->float->double chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { f = (float)x; x = (double)f * 1.0000001; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // fp64 sqrt chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // fp64 div chain
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // FFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = fmaf(f, 1.0001f, 1e-6f);
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
  // __syncthreads loop
  t0 = clock64();
  for (int i = 0; i < N; ++i) { __syncthreads(); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[8] = t1 - t0;
  out[threadIdx.x] = x + f;
}
__global__ void kthr(double *out, long long *cyc, int iters) {
  // DFMA throughput: 8 independent chains per thread, full block
  double a0=threadIdx.x,a1=a0+1,a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7; const double y=1.0000001;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a0=fma(a0,y,1e-9);a1=fma(a1,y,1e-9);a2=fma(a2,y,1e-9);a3=fma(a3,y,1e-9);a4=fma(a4,y,1e-9);a5=fma(a5,y,1e-9);a6=fma(a6,y,1e-9);a7=fma(a7,y,1e-9);}
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = t1 - t0;
  out[threadIdx.x] = a0+a1+a2+a3+a4+a5+a6+a7;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 0.5); k<<<1, 32>>>(o, c, 0.5);
  long long h[16]; cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char *nm[] = {"DFMA", "DMUL", "SHFL.f64", "LDS.64+cvt", "F2F f64<->f32", "sqrt f64", "div f64", "FFMA", "syncthreads(1 warp)"};
  for (int i = 0; i < 9; ++i) printf("%-22s %7.1f cycles\n", nm[i], (double)h[i] / N);
  int iters = 4096;
  kthr<<<1, 1024>>>(o, c, iters); kthr<<<1, 1024>>>(o, c, iters);
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  printf("DFMA throughput per SM: %.1f FMA/clk\n", 1024.0 * 8 * iters / h[9]);
  return 0;
}
