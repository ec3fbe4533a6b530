// Latency probes for the K-EIG round chain (B200): dependent fp64 ops, fp64 MUFU
// approximations, LDS->use, BAR.RED.OR, the rot2 chain of eig2.cuh. One CTA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_approx(double x) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rcp_approx(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(double *out, long long *t, int reps, double seed) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  double x = seed + tid * 1e-9;
  long long t0, t1;
  // 1. dependent DFMA
  t0 = clock64();
  for (int i = 0; i < reps; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (tid == 0) t[0] = (t1 - t0) / reps;
  // 2. dependent DMUL
  t0 = clock64();
  for (int i = 0; i < reps; ++i) x = x * 1.0000001;
  t1 = clock64(); if (tid == 0) t[1] = (t1 - t0) / reps;
  // 3. MUFU rsqrt f64 chain
  t0 = clock64();
  for (int i = 0; i < reps; ++i) x = rsqrt_approx(x) + 0.5;
  t1 = clock64(); if (tid == 0) t[2] = (t1 - t0) / reps;
  // 4. MUFU rcp f64 chain
  t0 = clock64();
  for (int i = 0; i < reps; ++i) x = rcp_approx(x) + 0.5;
  t1 = clock64(); if (tid == 0) t[3] = (t1 - t0) / reps;
  // 5. LDS -> address chain
  int idx = tid & 7;
  t0 = clock64();
  for (int i = 0; i < reps; ++i) { double v = sm[idx]; idx = ((int)v) & 7; }
  t1 = clock64(); if (tid == 0) t[4] = (t1 - t0) / reps;
  // 6. BAR.RED.OR loop (all threads)
  int b = 0;
  t0 = clock64();
  for (int i = 0; i < reps; ++i) b = __syncthreads_or(b ^ (x > 1e300));
  t1 = clock64(); if (tid == 0) t[5] = (t1 - t0) / reps;
  // 7. STS -> BAR -> LDS round trip
  t0 = clock64();
  for (int i = 0; i < reps; ++i) { sm[(tid + i) & 1023] = x; __syncthreads(); x += sm[(tid + 1 + i) & 1023] * 1e-20; }
  t1 = clock64(); if (tid == 0) t[6] = (t1 - t0) / reps;
  // 8. rot2 chain (eig2.cuh), dependent through g
  double a = 1.0, d = 2.0, g = x * 1e-3, thr = 1e-300;
  t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    const double dd = d - a, g2 = 2.0 * g;
    const double h2 = fma(dd, dd, g2 * g2);
    double rh = rsqrt_approx(h2);
    rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
    const double den = fabs(dd) + h2 * rh;
    double rc = rcp_approx(den);
    rc = rc * fma(-den, rc, 2.0);
    const bool on = fabs(g) > thr;
    const double tt = on ? (dd >= 0.0 ? g2 : -g2) * rc : 0.0;
    const double y = fma(tt, tt, 1.0);
    double cs = rsqrt_approx(y);
    cs = cs * fma(-0.5 * y, cs * cs, 1.5);
    cs = cs * fma(-0.5 * y, cs * cs, 1.5);
    g = cs * tt * 1e-3 + 1e-5;
  }
  t1 = clock64(); if (tid == 0) t[7] = (t1 - t0) / reps;
  // 9. fp64 compare+select chain
  t0 = clock64();
  for (int i = 0; i < reps; ++i) x = (x > 0.5) ? x * 0.5 : x + 1.0;
  t1 = clock64(); if (tid == 0) t[8] = (t1 - t0) / reps;
  out[tid] = x + g + b + idx;
}
int main() {
  double *o; long long *t; cudaMalloc(&o, 8192); cudaMallocManaged(&t, 16 * 8);
  const char *nm[] = {"DFMA dep", "DMUL dep", "MUFU.RSQ64H+DADD", "MUFU.RCP64H+DADD", "LDS->addr", "BAR.RED.OR", "STS,BAR,LDS", "rot2 chain", "DSETP+sel chain"};
  for (int th : {32, 64, 416, 512}) {
    k<<<1, th>>>(o, t, 1000, 0.7); cudaDeviceSynchronize();
    k<<<1, th>>>(o, t, 1000, 0.7); cudaDeviceSynchronize();
    printf("threads %d:", th);
    for (int i = 0; i < 9; ++i) printf("  %s %lld", nm[i], t[i]);
    printf("\n");
  }
  return 0;
}
