// Round cost of the two-sided K-EIG2 round (eig2.cuh) in isolation, n = 10 and 55, with
// parts switched off by the template mask: 1 B-block update, 2 producer rot2, 4 V update,
// 8 barrier as __syncthreads_or (else __syncthreads).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_approx(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rcp_approx(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
struct Rot2 { double c, s, a, d; };
__device__ __forceinline__ Rot2 rot2(double a, double d, double g, double thr) {
  const double dd = d - a, g2 = 2.0 * g;
  const double h2 = fma(dd, dd, g2 * g2);
  double rh = rsqrt_approx(h2);
  rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
  const double den = fabs(dd) + h2 * rh;
  double rc = rcp_approx(den);
  rc = rc * fma(-den, rc, 2.0);
  const bool on = fabs(g) > thr;
  const double t = on ? (dd >= 0.0 ? g2 : -g2) * rc : 0.0;
  const double y = fma(t, t, 1.0);
  double cs = rsqrt_approx(y);
  cs = cs * fma(-0.5 * y, cs * cs, 1.5);
  cs = cs * fma(-0.5 * y, cs * cs, 1.5);
  Rot2 R; R.c = on ? cs : 1.0; R.s = on ? cs * t : 0.0; R.a = fma(-t, g, a); R.d = fma(t, g, d);
  return R;
}
__device__ __forceinline__ int rr_pos(int j, int r, int M) { if (j == 0) return 0; int t = j - 1 + r; if (t >= M) t -= M; return 1 + t; }
template <int MASK>
__global__ void k(int NP, int rounds, long long *out, double *sink) {
  extern __shared__ __align__(16) double sm[];
  const int H = NP / 2, M = NP - 1, ld = NP + 2;
  double *Bm = sm, *V = sm + NP * ld;
  Rot2 *rec = (Rot2 *)(V + NP * ld);
  unsigned short *sched = (unsigned short *)(rec + 2 * H);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < NP * ld; e += nt) { Bm[e] = 1e-3 * ((e * 7) % 13); V[e] = 1e-2 * ((e * 5) % 11); }
  for (int e = tid; e < M * H; e += nt) { const int r = e / H, P = e - r * H; sched[e] = (unsigned short)(rr_pos(P, r, M) | (rr_pos(M - P, r, M) << 8)); }
  for (int P = tid; P < 2 * H; P += nt) { rec[P].c = 0.99; rec[P].s = 0.01; rec[P].a = 1.0; rec[P].d = 2.0; }
  const int NB = H * (H + 1) / 2, nV = H * H;
  int bP[2], bQ[2], bprod[2], vI[2], vQ[2];
  for (int k = 0; k < 2; ++k) {
    const int t = tid + k * nt;
    bP[k] = -1; bQ[k] = 0; bprod[k] = 0;
    if (t < NB) { int P = 0, rem = t; while (rem >= H - P) { rem -= H - P; ++P; } const int Q = P + rem; bP[k] = P; bQ[k] = Q;
      if (P == 0 && Q == 1) bprod[k] |= 1; if (P == H - 2 && Q == H - 1) bprod[k] |= 2; if (Q == P + 2) bprod[k] |= 4; }
    vI[k] = -1; vQ[k] = 0; if (t < nV) { vI[k] = t % H; vQ[k] = t / H; }
  }
  __syncthreads();
  const double thr = 1e-300, thr2 = 0.0;
  int big = 1, r = 0;
  long long t0 = clock64();
  for (int rounds_ = 0; rounds_ < rounds; ++rounds_) {
    const Rot2 *rc = rec + (rounds_ & 1) * H;
    Rot2 *rn = rec + ((rounds_ + 1) & 1) * H;
    const unsigned short *sr = sched + r * H;
    int mybig = 0;
    if (MASK & 1) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (bP[k] < 0) continue;
      const int P = bP[k], Q = bQ[k];
      const unsigned fs1 = sr[P]; const int f1 = fs1 & 0xff, s1 = fs1 >> 8;
      const Rot2 R1 = rc[P];
      if (P == Q) { Bm[f1 * ld + f1] = R1.a; Bm[s1 * ld + s1] = R1.d; Bm[s1 * ld + f1] = 0.0; Bm[f1 * ld + s1] = 0.0; continue; }
      const unsigned fs2 = sr[Q]; const int f2 = fs2 & 0xff, s2 = fs2 >> 8;
      const Rot2 R2 = rc[Q];
      const double b00 = Bm[f2 * ld + f1], b01 = Bm[s2 * ld + f1], b10 = Bm[f2 * ld + s1], b11 = Bm[s2 * ld + s1];
      const double m00 = R2.c * b00 - R2.s * b01, m01 = R2.s * b00 + R2.c * b01;
      const double m10 = R2.c * b10 - R2.s * b11, m11 = R2.s * b10 + R2.c * b11;
      const double n00 = R1.c * m00 - R1.s * m10, n10 = R1.s * m00 + R1.c * m10;
      const double n01 = R1.c * m01 - R1.s * m11, n11 = R1.s * m01 + R1.c * m11;
      const int pr = bprod[k];
      if ((MASK & 2) && pr) {
        const bool sf = pr & 4, ff = pr & 1;
        const double pa = sf ? R2.a : ff ? R1.a : R2.d, pd = sf ? R1.d : ff ? R2.a : R1.d, pg = sf ? n10 : ff ? n00 : n11;
        Rot2 R = rot2(pa, pd, pg, thr);
        R.c = 0.99; R.s = 0.01 + 1e-30 * R.s; R.a = 1.0 + 1e-30 * R.a; R.d = 2.0;   // keep values bounded
        rn[sf ? P + 1 : ff ? 0 : H - 1] = R;
      }
      Bm[f2 * ld + f1] = n00; Bm[f1 * ld + f2] = n00; Bm[s2 * ld + f1] = n01; Bm[f1 * ld + s2] = n01;
      Bm[f2 * ld + s1] = n10; Bm[s1 * ld + f2] = n10; Bm[s2 * ld + s1] = n11; Bm[s1 * ld + s2] = n11;
      if (fma(n00, n00, fma(n01, n01, fma(n10, n10, n11 * n11))) > thr2) mybig = 1;
    }
    }
    if (MASK & 4) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (vI[k] < 0) continue;
      const int Q = vQ[k];
      const double c = rc[Q].c, sn = rc[Q].s;
      if (sn != 0.0) {
        const unsigned fs = sr[Q];
        double2 *vp = (double2 *)(V + (fs & 0xff) * ld + 2 * vI[k]);
        double2 *vq = (double2 *)(V + (fs >> 8) * ld + 2 * vI[k]);
        const double2 x = *vp, z = *vq;
        *vp = make_double2(c * x.x - sn * z.x, c * x.y - sn * z.y);
        *vq = make_double2(sn * x.x + c * z.x, sn * x.y + c * z.y);
      }
    }
    }
    if (MASK & 8) big = __syncthreads_or(mybig); else __syncthreads();
    r = (r + 1 == M) ? 0 : r + 1;
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
  if (big == 7) sink[tid] = Bm[tid] + V[tid];
}
template <int MASK> void run(int NP, int th) {
  long long *o; double *s; cudaMallocManaged(&o, 8); cudaMalloc(&s, 8192);
  const int H = NP / 2, ld = NP + 2;
  size_t smem = 8 * (2 * NP * ld) + 32 * 2 * H + 2 * (NP - 1) * H + 64;
  cudaFuncSetAttribute(k<MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<MASK><<<1, th, smem>>>(NP, 200, o, s); cudaDeviceSynchronize();
  k<MASK><<<1, th, smem>>>(NP, 2000, o, s); cudaDeviceSynchronize();
  printf("NP %d threads %d mask %2d: %lld cycles/round (%s)\n", NP, th, MASK, o[0], cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int NP : {10, 56}) {
    const int th = NP == 10 ? 64 : 416;
    run<15>(NP, th); run<13>(NP, th); run<9>(NP, th); run<11>(NP, th); run<12>(NP, th); run<8>(NP, th); run<0>(NP, th); run<7>(NP, th);
  }
}
