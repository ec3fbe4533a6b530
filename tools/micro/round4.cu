// One-sided Jacobi round cost (n = 55, G = 8 lanes per pair, 8 warps) for two shared-memory
// layouts: column stride LD = 55 with the plain circle-method slot order (k_eig as of
// round 1), and LD = 56 (== 8 mod 16) with a parity-matched slot order: the two pairs that
// share a half-warp read columns of different parity, so their 64 B windows fall in
// different halves of the 128 B bank space (no bank conflicts).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_approx(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rcp_approx(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

template <int LD>
__global__ void k(const unsigned short *gsched, long long *out, int rounds) {
  const int n = 55, H = 28, G = 8, EPL = 7;
  __shared__ double U[72 * 56];
  __shared__ double nrm[56];
  __shared__ unsigned short sched[55 * 28];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = lane / G, sub = lane % G;
  for (int e = tid; e < 56 * 56; e += blockDim.x) U[e] = (e % 7) * 0.01 + (e % 57 == 0 ? 3.0 : 0.0);
  for (int j = tid; j < 56; j += blockDim.x) nrm[j] = 9.0;
  for (int e = tid; e < 55 * 28; e += blockDim.x) sched[e] = gsched[e];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    const int r = it % 55;
    const int P = warp * 4 + grp;
    int p = 0, q = 0; bool valid = P < H;
    if (valid) { unsigned pq = sched[r * H + P]; p = pq & 0xff; q = pq >> 8; valid = p < n && q < n; }
    double *up = U + p * LD, *uq = U + q * LD;
    double xp[EPL], xq[EPL], g0 = 0, g1 = 0;
#pragma unroll
    for (int c = 0; c < EPL; ++c) {
      const int i = sub + G * c; const bool ok = valid && i < n;
      xp[c] = ok ? up[i] : 0.0; xq[c] = ok ? uq[i] : 0.0;
      if (c & 1) g1 += xp[c] * xq[c]; else g0 += xp[c] * xq[c];
    }
    double ga = g0 + g1;
    for (int o = 4; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
    const double al = valid ? nrm[p] : 1.0, be = valid ? nrm[q] : 1.0;
    double cs = 1.0, sn = 0.0;
    if (valid && ga != 0.0) {
      const double d = be - al, g2 = 2.0 * ga;
      const double h2 = fma(d, d, g2 * g2);
      double rh = rsqrt_approx(h2); rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
      const double den = fabs(d) + h2 * rh;
      double rc = rcp_approx(den); rc = rc * fma(-den, rc, 2.0);
      const double t = (d >= 0.0 ? g2 : -g2) * rc * 1e-3;
      const double t2v = t * t;
      cs = fma(t2v, fma(t2v, 0.375, -0.5), 1.0); sn = cs * t;
    }
    if (valid) {
#pragma unroll
      for (int c = 0; c < EPL; ++c) { const int i = sub + G * c; if (i < n) { up[i] = cs * xp[c] - sn * xq[c]; uq[i] = sn * xp[c] + cs * xq[c]; } }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
}


// LDS.128 variant: lane sub holds elements 2*(sub + G c), +1 of both columns, column stride LD
template <int LD, int G>
__global__ void kv(const unsigned short *gsched, long long *out, int rounds) {
  const int n = 55, H = 28, EPL = 56 / (2 * G), PPW = 32 / G;
  __shared__ __align__(16) double U[72 * 56];
  __shared__ double nrm[56];
  __shared__ unsigned short sched[55 * 28];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, grp = lane / G, sub = lane % G;
  for (int e = tid; e < 72 * 56; e += blockDim.x) U[e] = ((e % LD) < n) ? (e % 7) * 0.01 + (e % (LD + 1) == 0 ? 3.0 : 0.0) : 0.0;
  for (int j = tid; j < 56; j += blockDim.x) nrm[j] = 9.0;
  for (int e = tid; e < 55 * 28; e += blockDim.x) sched[e] = gsched[e];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    const int r = it % 55;
    for (int P0 = warp * PPW; P0 < H; P0 += (blockDim.x / 32) * PPW) {
      const int P = P0 + grp;
      int p = 0, q = 0; bool valid = P < H;
      if (valid) { unsigned pq = sched[r * H + P]; p = pq & 0xff; q = pq >> 8; valid = p < n && q < n; }
      double2 *up = (double2 *)(U + p * LD), *uq = (double2 *)(U + q * LD);
      double2 xp[EPL], xq[EPL];
      double g0 = 0, g1 = 0;
#pragma unroll
      for (int c = 0; c < EPL; ++c) {
        const int i = sub + G * c;
        xp[c] = valid ? up[i] : make_double2(0.0, 0.0); xq[c] = valid ? uq[i] : make_double2(0.0, 0.0);
        g0 += xp[c].x * xq[c].x; g1 += xp[c].y * xq[c].y;
      }
      double ga = g0 + g1;
      for (int o = G / 2; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
      const double al = valid ? nrm[p] : 1.0, be = valid ? nrm[q] : 1.0;
      double cs = 1.0, sn = 0.0;
      if (valid && ga != 0.0) {
        const double d = be - al, g2 = 2.0 * ga;
        const double h2 = fma(d, d, g2 * g2);
        double rh = rsqrt_approx(h2); rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
        const double den = fabs(d) + h2 * rh;
        double rc = rcp_approx(den); rc = rc * fma(-den, rc, 2.0);
        const double t = (d >= 0.0 ? g2 : -g2) * rc * 1e-3;
        const double t2v = t * t;
        cs = fma(t2v, fma(t2v, 0.375, -0.5), 1.0); sn = cs * t;
      }
      if (valid) {
#pragma unroll
        for (int c = 0; c < EPL; ++c) {
          const int i = sub + G * c;
          up[i] = make_double2(cs * xp[c].x - sn * xq[c].x, cs * xp[c].y - sn * xq[c].y);
          uq[i] = make_double2(sn * xp[c].x + cs * xq[c].x, sn * xp[c].y + cs * xq[c].y);
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / rounds;
}

static void circle(int r, int P, int &p, int &q) {
  const int NP = 56;
  auto pos = [&](int j) { if (j == 0) return 0; int t = j - 1 + r; if (t >= NP - 1) t -= NP - 1; return 1 + t; };
  p = pos(P); q = pos(NP - 1 - P); if (p > q) { int t = p; p = q; q = t; }
}

int main() {
  std::vector<unsigned short> plain(55 * 28), matched(55 * 28);
  for (int r = 0; r < 55; ++r) {
    std::vector<std::pair<int, int>> ee, oo, eo;
    for (int P = 0; P < 28; ++P) {
      int p, q; circle(r, P, p, q);
      plain[r * 28 + P] = p | (q << 8);
      if ((p & 1) == 0 && (q & 1) == 0) ee.push_back({p, q});
      else if ((p & 1) && (q & 1)) oo.push_back({p, q});
      else eo.push_back((p & 1) ? std::make_pair(q, p) : std::make_pair(p, q));   // first even
    }
    std::vector<std::pair<int, int>> slots;
    for (size_t i = 0; i < ee.size(); ++i) { slots.push_back(ee[i]); slots.push_back(oo[i]); }
    for (size_t i = 0; i + 1 < eo.size(); i += 2) { slots.push_back(eo[i]); slots.push_back({eo[i + 1].second, eo[i + 1].first}); }
    if (ee.size() != oo.size() || slots.size() != 28) { printf("bad round %d\n", r); return 1; }
    for (int P = 0; P < 28; ++P) matched[r * 28 + P] = slots[P].first | (slots[P].second << 8);
  }
  unsigned short *ds; long long *d, h;
  cudaMalloc(&ds, 55 * 28 * 2); cudaMalloc(&d, 8);
  const int lds[] = {55, 56, 57, 58, 60, 64, 72};
  for (int v = 0; v < 14; ++v) {
    cudaMemcpy(ds, (v & 1) ? matched.data() : plain.data(), 55 * 28 * 2, cudaMemcpyHostToDevice);
    const int ld = lds[v / 2];
    for (int rep = 0; rep < 2; ++rep) {
      switch (ld) {
        case 55: k<55><<<1, 256>>>(ds, d, 5500); break;
        case 56: k<56><<<1, 256>>>(ds, d, 5500); break;
        case 57: k<57><<<1, 256>>>(ds, d, 5500); break;
        case 58: k<58><<<1, 256>>>(ds, d, 5500); break;
        case 60: k<60><<<1, 256>>>(ds, d, 5500); break;
        case 64: k<64><<<1, 256>>>(ds, d, 5500); break;
        default: k<72><<<1, 256>>>(ds, d, 5500); break;
      }
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("LD %d schedule %-8s  %lld cycles/round\n", ld, (v & 1) ? "matched" : "plain", h);
  }
  cudaMemcpy(ds, plain.data(), 55 * 28 * 2, cudaMemcpyHostToDevice);
  const char *nm[] = {"v128 LD56 G8 256t", "v128 LD72 G8 256t", "v128 LD56 G4 256t", "v128 LD72 G4 256t", "v128 LD56 G4 128t", "v128 LD60 G4 128t"};
  for (int v = 0; v < 6; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (v) {
        case 0: kv<56, 8><<<1, 256>>>(ds, d, 5500); break;
        case 1: kv<72, 8><<<1, 256>>>(ds, d, 5500); break;
        case 2: kv<56, 4><<<1, 256>>>(ds, d, 5500); break;
        case 3: kv<72, 4><<<1, 256>>>(ds, d, 5500); break;
        case 4: kv<56, 4><<<1, 128>>>(ds, d, 5500); break;
        default: kv<60, 4><<<1, 128>>>(ds, d, 5500); break;
      }
    }
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s  %lld cycles/round\n", nm[v], h);
  }
  return 0;
}
