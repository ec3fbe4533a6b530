// Phase timing of one one-sided Jacobi round (n = 55, G = 8 lanes per pair, 8 warps),
// mirroring k_eig's loop body; clock64 stamps per phase, warp 0 lane 0 reports.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_sum8(double v) {
  for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double rsqrt_approx(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rcp_approx(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__global__ void k(long long *out, int rounds, int mode) {
  const int n = 55, NP = 56, H = 28, G = 8, EPL = 8;
  __shared__ double U[55 * 55];
  __shared__ double nrm[56];
  __shared__ unsigned short sched[55 * 28];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = lane / G, sub = lane % G;
  for (int e = tid; e < n * n; e += blockDim.x) U[e] = (e % 7) * 0.01 + (e % n == e / n ? 3.0 : 0.0);
  for (int j = tid; j < n; j += blockDim.x) nrm[j] = 9.0;
  for (int e = tid; e < 55 * 28; e += blockDim.x) {
    const int r = e / H, P = e - r * H;
    auto pos = [&](int j) { if (j == 0) return 0; int t = j - 1 + r; if (t >= NP - 1) t -= NP - 1; return 1 + t; };
    int p = pos(P), q = pos(NP - 1 - P); if (p > q) { int t = p; p = q; q = t; }
    sched[e] = p | (q << 8);
  }
  __syncthreads();
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  for (int it = 0; it < rounds; ++it) {
    const int r = it % 55;
    long long t0 = clock64();
    const int P = warp * 4 + grp;
    int p = 0, q = 0; bool valid = P < H;
    if (valid) { unsigned pq = sched[r * H + P]; p = pq & 0xff; q = pq >> 8; valid = q < n; }
    double *up = U + p * n, *uq = U + q * n;
    double xp[EPL], xq[EPL], g0 = 0, g1 = 0;
#pragma unroll
    for (int c = 0; c < EPL; ++c) {
      const int i = sub + G * c; const bool ok = valid && i < n;
      xp[c] = ok ? up[i] : 0.0; xq[c] = ok ? uq[i] : 0.0;
      if (c & 1) g1 += xp[c] * xq[c]; else g0 += xp[c] * xq[c];
    }
    double ga = g0 + g1;
    long long t1 = clock64();
    ga = warp_sum8(ga);
    long long t2 = clock64();
    const double al = valid ? nrm[p] : 1.0, be = valid ? nrm[q] : 1.0;
    double cs = 1.0, sn = 0.0;
    if (mode == 0 && valid && ga != 0.0) {
      const double d = be - al, g2 = 2.0 * ga;
      const double h2 = fma(d, d, g2 * g2);
      double rh = rsqrt_approx(h2); rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
      const double den = fabs(d) + h2 * rh;
      double rc = rcp_approx(den); rc = rc * fma(-den, rc, 2.0);
      const double t = (d >= 0.0 ? g2 : -g2) * rc * 1e-3;
      const double t2v = t * t;
      cs = fma(t2v, fma(t2v, 0.375, -0.5), 1.0); sn = cs * t;
    }
    long long t3 = clock64();
    if (valid) {
#pragma unroll
      for (int c = 0; c < EPL; ++c) { const int i = sub + G * c; if (i < n) { up[i] = cs * xp[c] - sn * xq[c]; uq[i] = sn * xp[c] + cs * xq[c]; } }
    }
    long long t4 = clock64();
    __syncthreads();
    long long t5 = clock64();
    acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3; acc[4] += t5 - t4; acc[5] += t5 - t0;
  }
  if (tid == 0) for (int k = 0; k < 6; ++k) out[k] = acc[k] / rounds;
  if (tid == 32 * 6) for (int k = 0; k < 6; ++k) out[6 + k] = acc[k] / rounds;
}
int main() {
  long long *d, h[12];
  cudaMalloc(&d, 12 * 8);
  const char *nm[] = {"load+dot", "shuffle", "rotation", "apply", "barrier", "round total"};
  for (int mode = 0; mode < 2; ++mode)
    for (int threads : {256, 224}) {
      k<<<1, threads>>>(d, 550, mode); k<<<1, threads>>>(d, 5500, mode);
      cudaMemcpy(h, d, 12 * 8, cudaMemcpyDeviceToHost);
      printf("mode %d (rotation %s) threads %d\n", mode, mode == 0 ? "on" : "off", threads);
      for (int i = 0; i < 6; ++i) printf("  %-12s warp0 %6lld  warp6 %6lld cycles\n", nm[i], h[i], h[6 + i]);
    }
  return 0;
}
