// Progressive cost of a Jacobi round's pieces (n = 55 columns of stride 56 in shared
// memory, 8 lanes per pair, 7 warps): A loads+dot, B +shuffle reduce, C +rotation math,
// D +stores (= full round), E = D without the barrier (race, timing only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_approx(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rcp_approx(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ void cs64(double al, double be, double ga, double &cs, double &sn) {
  const double d = be - al, g2 = 2.0 * ga;
  const double h2 = fma(d, d, g2 * g2);
  double rh = rsqrt_approx(h2); rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
  const double den = fabs(d) + h2 * rh;
  double rc = rcp_approx(den); rc = rc * fma(-den, rc, 2.0);
  const double t = (d >= 0.0 ? g2 : -g2) * rc;
  const double t2 = t * t;
  cs = fma(t2, fma(t2, 0.375, -0.5), 1.0);
  sn = cs * t;
}
template <int V>
__global__ void k(long long *out, int rounds, const unsigned short *gsched) {
  constexpr int n = 55, H = 28, LD = 56;
  __shared__ __align__(16) double U[56 * 56];
  __shared__ unsigned short sched[55 * 28];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = lane / 8, sub = lane % 8;
  for (int e = tid; e < 56 * 56; e += blockDim.x) U[e] = 1e-3 * (e % 13) + ((e % 57) == 0 ? 3.0 : 0.0);
  for (int e = tid; e < 55 * 28; e += blockDim.x) sched[e] = gsched[e];
  __syncthreads();
  const int P = warp * 4 + grp;
  const int nwarps = blockDim.x >> 5;
  __shared__ int prog[32];
  if (tid < 32) prog[tid] = 0;
  __syncthreads();
  double sink = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    const int r = it % 55;
    if (V == 5 && it > 0) {   // wait for the neighbouring warps to finish round it - 1
      if (lane == 0) {
        const volatile int *pv = prog;
        while ((warp > 0 && pv[warp - 1] < it) || (warp + 1 < nwarps && pv[warp + 1] < it)) {}
        __threadfence_block();
      }
      __syncwarp();
    }
    int p = 0, q = 1;
    if (P < H) { const unsigned pq = sched[r * H + P]; p = pq & 0xff; q = pq >> 8; if (q >= n) q = n - 1; }
    double *up = U + p * LD, *uq = U + q * LD;
    double xp[8], xq[8], g0 = 0, g1 = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 2 * sub + 16 * c;
      const double2 a = *(const double2 *)(up + i), b = *(const double2 *)(uq + i);
      xp[2 * c] = a.x; xp[2 * c + 1] = a.y; xq[2 * c] = b.x; xq[2 * c + 1] = b.y;
      g0 += a.x * b.x; g1 += a.y * b.y;
    }
    double ga = g0 + g1;
    if (V >= 1) {
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
    }
    double cs = 1.0, sn = 1e-9 * ga;
    if (V >= 2) cs64(xp[0] * xp[0] + 1.0, xq[1] * xq[1] + 2.0, ga * 1e-3, cs, sn);
    if (V >= 3 && P < H) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 2 * sub + 16 * c;
        *(double2 *)(up + i) = make_double2(cs * xp[2 * c] - sn * xq[2 * c], cs * xp[2 * c + 1] - sn * xq[2 * c + 1]);
        *(double2 *)(uq + i) = make_double2(sn * xp[2 * c] + cs * xq[2 * c], sn * xp[2 * c + 1] + cs * xq[2 * c + 1]);
      }
    } else {
      sink += cs + sn;
    }
    if (V == 5) {
      __syncwarp();
      if (lane == 0) { __threadfence_block(); ((volatile int *)prog)[warp] = it + 1; }
    } else if (V != 4) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  if (sink == 12345.0) out[1] = 1;
}
int main() {
  unsigned short hs[55 * 28];
  auto pos = [](int j, int r) { if (j == 0) return 0; int t = j - 1 + r; if (t >= 55) t -= 55; return 1 + t; };
  for (int r = 0; r < 55; ++r)
    for (int P = 0; P < 28; ++P) { int p = pos(P, r), q = pos(55 - P, r); if (p > q) { int t = p; p = q; q = t; } hs[r * 28 + P] = p | (q << 8); }
  unsigned short *ds; cudaMalloc(&ds, sizeof(hs)); cudaMemcpy(ds, hs, sizeof(hs), cudaMemcpyHostToDevice);
  long long *d, h; cudaMalloc(&d, 16);
  auto run = [&](auto kern, const char *name, int threads) {
    kern<<<1, threads>>>(d, 550, ds); kern<<<1, threads>>>(d, 5500, ds);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-44s threads %d: %lld cycles/round\n", name, threads, h);
  };
  for (int th : {224, 256}) {
    run(k<0>, "A loads + dot + barrier", th);
    run(k<1>, "B A + shuffle reduce", th);
    run(k<2>, "C B + rotation math", th);
    run(k<3>, "D C + stores (full round)", th);
    run(k<4>, "E D without barrier", th);
    run(k<5>, "F D with neighbour-warp flags", th);
  }
  return 0;
}
