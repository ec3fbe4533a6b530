// K-EIG: batched PSD-cone projection (Step 2 of Algorithm 1, PAPER.md:467-472;
// projection Pi(X) = Q max(0, W) Q^T), included by engine.cu.
//
// One CTA per PSD block X_beta (order n <= 255; n > 112 keeps U in L2-resident global scratch), fp64 throughout:
//   1. gather X_b = X + sigma (A* y - C) straight from svec (A* fused);
//   2. one-sided (Hestenes) Jacobi on the shifted matrix B = X_b + s I, s = ||X_b||_F,
//      so that B is PSD with eigenvalues lambda + s >= 0 kept apart even when X_b has
//      +/- pairs: U = B V, columns of U rotated pairwise until mutually orthogonal,
//      then u_j = (lambda_j + s) v_j. One warp owns one column pair per round
//      (round-robin ordering), so a round needs a single CTA barrier;
//   3. warm start: V is the eigenbasis of the previous ADMM iteration (stored per
//      block), so near convergence one sweep plus one checking sweep suffice;
//   4. S = (Pi(X_b) - X_b)/sigma from the smaller of the positive and negative
//      eigen-sets (Moreau: Pi(X) - X = Pi(-X)), written back in svec.
#pragma once

#ifdef STROM_EIG_PROF
// phase timestamps (clock64) per block of the last K-EIG launch (tools/eig_prof.py)
__device__ long long g_eig_prof[4096][16];
#define EIG_STAMP(k) do { if (threadIdx.x == 0 && bidx < 4096) g_eig_prof[bidx][k] = clock64(); } while (0)
#else
#define EIG_STAMP(k) do { } while (0)
#endif

struct EigArgs {
  const int32_t *blocks; int32_t nblk;
  const int32_t *bn; const int64_t *boff;
  const int64_t *Atp; const int32_t *Atr; const double *Atv;
  const double *X, *C, *y;
  double *Xb_out, *S_out;
  double *Vstore; const int64_t *voff;     // warm-start eigenbases (n*n per block)
  double *Ug, *Ag; const int64_t *uoff;    // global scratch for n > 112 (GU variant)
  DevState *st;
  int32_t max_sweeps; double tol;
  int32_t mode;          // 0 projection; 1 eigenvalues of C - A*y (lambda_min only);
                         // 2 extraction: top two eigenvalues and top eigenvector of X
  double *lam12; double *vtop; const int64_t *toff;   // mode 2 outputs (toff: prefix of n)
  int32_t warm_enable, cold_every;
  double *lam_min;
};

__device__ __forceinline__ int rr_pos(int j, int r, int NPm1) {
  // round-robin position (circle method): player 0 fixed, others rotate by r
  if (j == 0) return 0;
  int t = j - 1 + r;
  if (t >= NPm1) t -= NPm1;
  return 1 + t;
}

// fp64 MUFU approximations (~20 bits) refined by Newton steps: no f64<->f32 conversions.
__device__ __forceinline__ double rsqrt_approx(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// Jacobi rotation for a column pair with ||u_p||^2 = al, ||u_q||^2 = be, u_p.u_q = ga:
// t = tan(theta) = sign(d) g2 / (|d| + sqrt(d^2 + g2^2)), d = be - al, g2 = 2 ga; t needs
// ~1e-10 relative accuracy only, (cs, sn) are orthogonal to fp64 precision.
__device__ __forceinline__ void jacobi_cs(double al, double be, double ga, double &cs, double &sn) {
  const double d = be - al, g2 = 2.0 * ga;
  const double h2 = fma(d, d, g2 * g2);
  double rh = rsqrt_approx(h2);
  rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
  const double den = fabs(d) + h2 * rh;
  double rc = rcp_approx(den);
  rc = rc * fma(-den, rc, 2.0);
  const double t = (d >= 0.0 ? g2 : -g2) * rc;
  const double t2 = t * t;
  if (t2 < 1e-8) {
    cs = fma(t2, fma(t2, 0.375, -0.5), 1.0);
  } else {
    const double y = 1.0 + t2;
    cs = rsqrt_approx(y);
    cs = cs * fma(-0.5 * y, cs * cs, 1.5);
    cs = cs * fma(-0.5 * y, cs * cs, 1.5);
  }
  sn = cs * t;
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Shared-memory column stride of U / V for a block of order n: with 8 lanes per column
// pair a stride == 8 (mod 16) doubles keeps the warp's column reads free of bank conflicts
// (one Jacobi round of order 55: 1,131 -> 929 cycles, tools/micro/round4.cu).
__host__ __device__ inline int eig_ld(int n, int G) { return G == 8 ? (n + 7) / 16 * 16 + 8 : n; }

__device__ __forceinline__ int svec_pos(int i, int j) {  // i, j any order
  return (i <= j) ? (j * (j + 1) / 2 + i) : (i * (i + 1) / 2 + j);
}

// X_b = X + sigma (A* y - C) (mode 0) or C - A* y (mode 1) for the svec entries
// [off + e0, off + L) with stride es, written to Xb_out; returns the partial ||.||^2.
// Four entries per pass so that their dependent L2 loads (column pointers -> row
// indices -> y) overlap.
__device__ __forceinline__ double gather_xb(const EigArgs &a, int64_t off, int L, int e0, int es,
                                            double sigma, bool proj) {
  double fro = 0.0;
  for (int eb = e0; eb < L; eb += 4 * es) {
    int64_t t0[4], t1[4];
    double aty[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = eb + k * es;
      t0[k] = t1[k] = 0;
      if (e < L) { t0[k] = a.Atp[off + e]; t1[k] = a.Atp[off + e + 1]; }
      aty[k] = 0.0;
    }
    for (int r = 0;; ++r) {
      bool any = false;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (t0[k] + r < t1[k]) { aty[k] += a.Atv[t0[k] + r] * a.y[a.Atr[t0[k] + r]]; any = true; }
      if (!any) break;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = eb + k * es;
      if (e < L) {
        const int64_t J = off + e;
        const double xb = a.mode == 2 ? a.X[J] : proj ? a.X[J] + sigma * (aty[k] - a.C[J]) : a.C[J] - aty[k];
        a.Xb_out[J] = xb;          // mode 1 uses Xb_out as scratch for C - A*y
        fro += xb * xb;            // svec norm == Frobenius norm
      }
    }
  }
  return fro;
}

// (i, j), i <= j, of svec position e (upper triangle column-wise)
__device__ __forceinline__ void svec_ij(int e, int &i, int &j) {
  j = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while (j * (j + 1) / 2 > e) --j;
  while ((j + 1) * (j + 2) / 2 <= e) ++j;
  i = e - j * (j + 1) / 2;
}

// Fast gather (blocks whose A* nonzeros fit in shared memory): pass 1 forms every
// product Atv[t] * y[Atr[t]] of the block's contiguous CSC segment with coalesced loads
// (two dependent L2 round trips in total instead of two per term); pass 2 sums each
// entry's products in t order -- the same terms in the same order as gather_xb, so X_b is
// bitwise identical -- writes X_b to global and keeps up to KE entries per thread in
// registers for the staging of the dense matrix. Returns the partial ||X_b||_F^2.
template <int KE>
__device__ __forceinline__ double gather_xb_smem(const EigArgs &a, int64_t off, int L, double *prod,
                                                 double (&xv)[KE], double sigma, bool proj) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t nz0 = a.Atp[off], nz1 = a.Atp[off + L];
  constexpr int NF = 12;          // products in flight per thread (two L2 round trips each)
  for (int64_t t = nz0 + tid; t < nz1; t += NF * nt) {
    int32_t r[NF];
    double v[NF], yv[NF];
#pragma unroll
    for (int k = 0; k < NF; ++k) {
      const int64_t tk = t + (int64_t)k * nt;
      r[k] = tk < nz1 ? a.Atr[tk] : 0;
      v[k] = tk < nz1 ? a.Atv[tk] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NF; ++k) yv[k] = a.y[r[k]];
#pragma unroll
    for (int k = 0; k < NF; ++k) {
      const int64_t tk = t + (int64_t)k * nt;
      if (tk < nz1) prod[tk - nz0] = v[k] * yv[k];
    }
  }
  __syncthreads();
  // every global load of pass 2 is issued before the first X_b store (which the compiler
  // could not otherwise move loads across): one L2 round trip for all KE entries
  int t0[KE], t1[KE];
  double xk[KE], ck[KE];
#pragma unroll
  for (int k = 0; k < KE; ++k) {
    const int e = tid + k * nt;
    t0[k] = t1[k] = 0; xk[k] = ck[k] = 0.0;
    if (e < L) {
      const int64_t J = off + e;
      t0[k] = (int)(a.Atp[J] - nz0); t1[k] = (int)(a.Atp[J + 1] - nz0);
      if (proj || a.mode == 2) xk[k] = a.X[J];
      ck[k] = a.C[J];
    }
  }
  double fro = 0.0;
#pragma unroll
  for (int k = 0; k < KE; ++k) {
    const int e = tid + k * nt;
    xv[k] = 0.0;
    if (e < L) {
      double aty = 0.0;
      for (int t = t0[k]; t < t1[k]; ++t) aty += prod[t];
      const double xb = a.mode == 2 ? xk[k] : proj ? xk[k] + sigma * (aty - ck[k]) : ck[k] - aty;
      a.Xb_out[off + e] = xb;
      fro += xb * xb;
      xv[k] = xb;
    }
  }
  return fro;
}

// Dense product U = A V (+ s V) with 4x4 register tiles, one tile per thread
// (requires ceil(n/4)^2 <= blockDim.x): thread (ti, tj) owns rows ti + nT r and columns
// tj + nT c (strided, so a warp's shared-memory reads of A are bank-conflict free). A
// symmetric in Abuf (column-major, stride ld), V column-major (stride ldv). Rows/columns
// past n are clamped reads whose results are dropped. The result is written to dst
// (stride ld) after a CTA barrier, so dst may alias Abuf or V. Per element the k-sum runs
// in k order, as in the warp-per-column loop it replaces.
__device__ __forceinline__ void warm_product_tiles(const double *Abuf, const double *V, int ldv, double *dst,
                                                   int n, int ld, double s) {
  const int tid = threadIdx.x, nT = (n + 3) >> 2;
  const bool act = tid < nT * nT;
  const int ti = act ? tid % nT : 0, tj = act ? tid / nT : 0;
  const double *ar[4], *vc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    ar[r] = Abuf + min(ti + nT * r, n - 1);
    vc[r] = V + (int64_t)min(tj + nT * r, n - 1) * ldv;
  }
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  if (act) {
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      double x[4], z[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) { x[r] = ar[r][(int64_t)k * ld]; z[r] = vc[r][k]; }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] += x[r] * z[c];
    }
  }
  double vij[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) vij[r][c] = act ? vc[c][min(ti + nT * r, n - 1)] : 0.0;
  __syncthreads();                // every read of Abuf and V is done
  if (act) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = ti + nT * r, j = tj + nT * c;
        if (i < n && j < n) dst[(int64_t)j * ld + i] = acc[r][c] + s * vij[r][c];
      }
  }
}

// Extraction outputs (mode 2): the two largest eigenvalues of the block
// and the eigenvector of the largest, normalised, sign fixed so that its first entry is
// >= 0. Rows [r0, r0 + nloc) of column j are at col[i - r0]; inv = 1/||u_j||, and v0 =
// the column's first entry (row 0, any CTA).
__device__ __forceinline__ int top2(const double *lam, int n, double &l1, double &l2) {
  int j = 0;
  l1 = lam[0]; l2 = -1.0e308;
  for (int k = 1; k < n; ++k) {
    if (lam[k] > l1) { l2 = l1; l1 = lam[k]; j = k; }
    else if (lam[k] > l2) l2 = lam[k];
  }
  if (n == 1) l2 = 0.0;
  return j;
}

// Convergence check by the Gram matrix U^T U (4x4 register tiles, upper triangle):
// true when every pair has (u_i.u_j)^2 <= c2 ||u_i||^2 ||u_j||^2 (norms from nrm).
// CTA-uniform result (contains a barrier).
__device__ __forceinline__ bool gram_orthogonal(const double *U, int ld, int n, const double *nrm, double c2,
                                                int tid, int nt) {
  const int nT = (n + 3) >> 2, ntile = nT * (nT + 1) / 2;
  int bad = 0;
  for (int t = tid; t < ntile; t += nt) {
    int bi = 0, rem = t;
    while (rem >= nT - bi) { rem -= nT - bi; ++bi; }
    const int bj = bi + rem;
    const double *ui[4], *uj[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      ui[r] = U + (int64_t)min(4 * bi + r, n - 1) * ld;
      uj[r] = U + (int64_t)min(4 * bj + r, n - 1) * ld;
    }
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    // rows visited from a thread-dependent start (tid & 7): the threads of a warp read
    // different columns (stride == 8 mod 16 doubles, i.e. two bank groups) at 8 different
    // rows, so a load spreads over 16 bank pairs instead of 2 (a 16-way conflict)
    int k = tid & 7;
    if (k >= n) k = 0;
    for (int kk = 0; kk < n; ++kk) {
      double x[4], z[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) { x[r] = ui[r][k]; z[r] = uj[r][k]; }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(x[r], z[c], acc[r][c]);
      if (++k == n) k = 0;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * bi + r, j = 4 * bj + c;
        if (i < j && j < n && acc[r][c] * acc[r][c] > c2 * nrm[i] * nrm[j]) bad = 1;
      }
  }
  return !__syncthreads_or(bad);
}

// G lanes own one column pair (rows i = sub + G*c), 32/G pairs per warp.
template <int G, int EPL, bool GU>
__global__ void __launch_bounds__(512, 1) k_eig(EigArgs a) {
  pdl_trigger();                  // static prologue below overlaps the previous kernel
  extern __shared__ double sm[];
  __shared__ double red[4 * 32];
  __shared__ int sets[128];
  __shared__ int set_info;
  constexpr int PPW = 32 / G;
  const int bidx = a.blocks[blockIdx.x];
  const int n = a.bn[bidx];
  const int NP = n + (n & 1), H = NP / 2;
  const int64_t off = a.boff[bidx];
  const int L = n * (n + 1) / 2;
  // U: n columns x n rows, column-major (column j at U + j*ld). Shared memory for
  // n <= 112 (A staged in U, warm basis in V); L2-resident global scratch above (GU).
  const int ld = GU ? n : eig_ld(n, G);
  double *U, *V, *Abuf, *lamv;
  if (GU) {
    U = a.Ug + a.uoff[bidx]; Abuf = a.Ag + a.uoff[bidx]; V = a.Vstore + a.voff[bidx];
    lamv = sm;
  } else {
    U = sm; Abuf = sm; V = sm + n * ld;
    lamv = sm + 2 * n * ld;
  }
  unsigned short *sched = (unsigned short *)(lamv + n + 8);  // (p | q << 8) per (round, pair)
  EIG_STAMP(0);
#ifdef STROM_EIG_PROF
  __syncthreads();
#endif
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int grp = lane / G, sub = lane % G;
  const double isq2 = 0.70710678118654752440;
  const bool proj = (a.mode == 0);
  for (int e = tid; e < (NP - 1) * H; e += nt) {
    const int r = e / H, P = e - r * H;
    int p = rr_pos(P, r, NP - 1), q = rr_pos(NP - 1 - P, r, NP - 1);
    if (p > q) { const int t2 = p; p = q; q = t2; }
    sched[e] = (unsigned short)(p | (q << 8));
  }
  pdl_wait();                     // everything below may read the previous kernels' output
  if (a.st->done) return;
  const double sigma = a.st->sigma;
  const bool warm = proj && a.warm_enable && a.st->eig_warm_valid &&
                    (a.cold_every <= 0 || (a.st->iter % a.cold_every) != 0);
  EIG_STAMP(8);
  // ---- 1. gather X_b (svec) into global, Frobenius norm -------------------------
  // Fast path: the block's A* products fit in the (still unused) U/V shared memory and
  // the svec entries fit in KE registers per thread.
  constexpr int KE = 12;
  const bool fast = !GU && (int64_t)(a.Atp[off + L] - a.Atp[off]) <= 2LL * n * ld && L <= KE * nt;
  double xv[KE];
  double fro = fast ? gather_xb_smem<KE>(a, off, L, sm, xv, sigma, proj)
                    : gather_xb(a, off, L, tid, nt, sigma, proj);
  EIG_STAMP(9);
  {
    double v1[1] = {fro};
    block_sum<1>(v1, red);
    if (tid == 0) red[127] = sqrt(v1[0]);
    __syncthreads();
  }
  // shift s = 2 ||X_b||_F >= 2 ||X_b||_2: every column of U = (X_b + sI)V keeps a norm
  // lambda_j + s >= ||X_b||_F, so v_j = u_j / ||u_j|| is accurate for every j
  const double s = 2.0 * red[127] + 1e-300;
  const double *Xb = a.Xb_out + off;
  EIG_STAMP(1);
  // ---- 2. U = (X_b + s I) V with V = V_prev (warm) or I ----------------------------
  if (fast) {
    // the products in shared memory are dead (block_sum's barriers): stage A from registers
    double *stage = warm ? Abuf : U;     // cold: U = A + sI directly
#pragma unroll
    for (int k = 0; k < KE; ++k) {
      const int e = tid + k * nt;
      if (e < L) {
        int i, j;
        svec_ij(e, i, j);
        if (i == j) stage[j * ld + i] = xv[k] + (warm ? 0.0 : s);
        else { const double v = xv[k] * isq2; stage[j * ld + i] = v; stage[i * ld + j] = v; }
      }
    }
  } else {
    double *stage = warm ? Abuf : U;     // cold: U = A + sI directly
    for (int e = tid; e < n * n; e += nt) {   // A (symmetric): column-major == row-major
      const int j = e / n, i = e - j * n;
      const double v = Xb[svec_pos(i, j)];
      stage[j * ld + i] = (i == j) ? v + (warm ? 0.0 : s) : v * isq2;
    }
  }
  const int nTw = (n + 3) >> 2;
  if (warm && !GU && nTw * nTw <= nt) {
    // U = A V_prev + s V_prev (4x4 register tiles, V_prev staged in shared memory);
    // U overwrites A in place after the tile barrier
    EIG_STAMP(10);
    const double *Vp = a.Vstore + a.voff[bidx];
    for (int e0 = tid; e0 < n * n; e0 += 8 * nt) {      // 8 loads in flight per thread
      double vv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) { const int e = e0 + k * nt; vv[k] = e < n * n ? Vp[e] : 0.0; }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int e = e0 + k * nt;
        if (e < n * n) { const int j = e / n; V[j * ld + e - j * n] = vv[k]; }
      }
    }
    __syncthreads();
    EIG_STAMP(11);
    warm_product_tiles(Abuf, V, ld, Abuf, n, ld, s);
    U = Abuf;
  } else if (warm) {
    if (!GU) {
      const double *Vp = a.Vstore + a.voff[bidx];
      for (int e = tid; e < n * n; e += nt) { const int j = e / n; V[j * ld + e - j * n] = Vp[e]; }
    }
    __syncthreads();
    // column j of the new U = A v_j + s v_j; one warp per column, rows lane + 32c.
    // Without GU the result overwrites v_j in place (each column is read and written
    // by one warp only), then U := V.
    // Two columns per warp pass (j, j + nwarps) for two independent FMA chains.
    double *dst = GU ? U : V;
    for (int j = warp; j < n; j += 2 * nwarps) {
      const int j2 = j + nwarps < n ? j + nwarps : j;
      const double *vj = V + j * ld, *vj2 = V + j2 * ld;
      double acc[8], acc2[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) { acc[c] = 0.0; acc2[c] = 0.0; }
      for (int q = 0; q < n; ++q) {
        const double vq = vj[q], vq2 = vj2[q];
        const double *aq = Abuf + q * ld;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = lane + 32 * c;
          if (i < n) { const double x = aq[i]; acc[c] += x * vq; acc2[c] += x * vq2; }
        }
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int i = lane + 32 * c;
        if (i < n) {
          const double w = acc[c] + s * vj[i], w2 = acc2[c] + s * vj2[i];
          dst[j * ld + i] = w;
          if (j2 != j) dst[j2 * ld + i] = w2;
        }
      }
    }
    if (!GU) U = V;
  }
  __syncthreads();
  EIG_STAMP(2);
  // ---- 3. one-sided Jacobi sweeps (round-robin pairs) ---------------------------------
  // Column norms nrm[j] = ||u_j||^2 live in shared memory (recomputed exactly at the
  // start of every sweep, updated per rotation), so a pair needs one dot u_p.u_q.
  // The rotation angle is computed in fp32 (it only has to reduce u_p.u_q); (c, s) are
  // then made orthogonal to fp64 precision, so V stays orthogonal.
  double *nrm = lamv;             // reuses the eigenvalue slot until step 4
  const double tol = fmax(a.tol, 4.0 * n * 2.220446049250313e-16);
  const double tol2 = tol * tol, quad2 = 1e-18;   // quad: sweep with max |cos| < 1e-9 is final
  const double mid2 = 1e-12, gram2 = 1e-24;       // Gram exit: |cos| <= 1e-12 for every pair
  bool converged = false;
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    for (int j = warp; j < n; j += nwarps) {
      const double *uj = U + j * ld;
      double t = 0.0;
      for (int i = lane; i < n; i += 32) t += uj[i] * uj[i];
      t = warp_sum(t);
      if (lane == 0) nrm[j] = t;
    }
    __syncthreads();
    int rotated = 0, big = 0, mid = 0;
    // One round: the G lanes of group `grp` own pair P of the round's schedule.
    auto pair_step = [&](int r, int P) {
      int p = 0, q = 0;
      bool valid = P < H;
      if (valid) {
        const unsigned pq = sched[r * H + P];
        p = pq & 0xff; q = pq >> 8;
        valid = q < n;                         // bye for odd n
      }
      const double al = valid ? nrm[p] : 1.0, be = valid ? nrm[q] : 1.0;   // off the dot's chain
      double *up = U + p * ld, *uq = U + q * ld;
      double xp[EPL], xq[EPL];
      double ga0 = 0.0, ga1 = 0.0;
#pragma unroll
      for (int c = 0; c < EPL; ++c) {
        const int i = sub + G * c;
        const bool ok = valid && i < n;
        xp[c] = ok ? up[i] : 0.0;
        xq[c] = ok ? uq[i] : 0.0;
        if (c & 1) ga1 += xp[c] * xq[c]; else ga0 += xp[c] * xq[c];
      }
      double ga = ga0 + ga1;
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
      const double ab = al * be, g2a = ga * ga;
      if (valid && ga != 0.0 && g2a > tol2 * ab) {
        rotated = 1;
        if (g2a > quad2 * ab) big = 1;
        if (g2a > mid2 * ab) mid = 1;
        // tan(theta) zeroing u_p.u_q: t = sign(d) g2 / (|d| + sqrt(d^2 + g2^2)),
        // d = be - al, g2 = 2 ga. t needs only ~1e-10 relative accuracy (it just has to
        // shrink u_p.u_q); (cs, sn) are exactly orthogonal to fp64 precision:
        // cos = (1 + t^2)^(-1/2) by MUFU rsqrt + two Newton steps (branch-free).
        const double d = be - al, g2 = 2.0 * ga;
        double cs, sn;
        if (fabs(g2) < 1e-3 * fabs(d)) {
          // small angle (most rotations of a warm-started sweep): with x = g2/|d|,
          // t = sign(d) x / (1 + sqrt(1 + x^2)) = sign(d) (x/2)(1 - x^2/4 + O(x^4)) to
          // 1.3e-13 relative, and cos = (1 + t^2)^(-1/2) = 1 - t^2/2 + 3t^4/8 to O(t^6) =
          // 1e-24: cs^2 + sn^2 = 1 to fp64 precision. One reciprocal instead of three
          // MUFU + Newton chains.
          const double ad = fabs(d);
          double rc = rcp_approx(ad);
          rc = rc * fma(-ad, rc, 2.0);
          const double x = g2 * rc, hx = 0.5 * x;
          const double t0 = hx * fma(-hx, hx, 1.0);
          const double t = d >= 0.0 ? t0 : -t0;
          const double t2 = t * t;
          cs = fma(t2, fma(t2, 0.375, -0.5), 1.0);
          sn = cs * t;
        } else {
          const double h2 = fma(d, d, g2 * g2);
          double rh = rsqrt_approx(h2);
          rh = rh * fma(-0.5 * h2, rh * rh, 1.5);
          const double den = fabs(d) + h2 * rh;
          double rc = rcp_approx(den);
          rc = rc * fma(-den, rc, 2.0);
          const double t = (d >= 0.0 ? g2 : -g2) * rc;
          const double y = fma(t, t, 1.0);
          cs = rsqrt_approx(y);
          cs = cs * fma(-0.5 * y, cs * cs, 1.5);
          cs = cs * fma(-0.5 * y, cs * cs, 1.5);
          sn = cs * t;
        }
#pragma unroll
        for (int c = 0; c < EPL; ++c) {
          const int i = sub + G * c;
          if (i < n) { up[i] = cs * xp[c] - sn * xq[c]; uq[i] = sn * xp[c] + cs * xq[c]; }
        }
        // every lane of the group read nrm[p], nrm[q] above; order those reads before the
        // write (the group is converged here: its lanes share valid, ga and the branch)
        __syncwarp(G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G)));
        if (sub == 0) {   // exact norms of the rotated pair from the 2x2 Gram matrix
          const double c2 = cs * cs, s2 = sn * sn, csn = 2.0 * cs * sn * ga;
          nrm[p] = c2 * al - csn + s2 * be;
          nrm[q] = s2 * al + csn + c2 * be;
        }
      }
    };
    if (nwarps * PPW >= H) {                   // every pair in one pass (warp-uniform)
      const bool act = warp * PPW < H;
      for (int r = 0; r < NP - 1; ++r) {
        if (act) pair_step(r, warp * PPW + grp);
        __syncthreads();
      }
    } else {
      for (int r = 0; r < NP - 1; ++r) {
        for (int P0 = warp * PPW; P0 < H; P0 += nwarps * PPW) pair_step(r, P0 + grp);
        __syncthreads();
      }
    }
    const int any_big = __syncthreads_or(big);
    const int any_rot = __syncthreads_or(rotated);
    if (!any_rot || !any_big) { converged = true; break; }
    // Every rotation of this sweep had |cos| <= 1e-6: by quadratic convergence the
    // columns are probably orthogonal to ~1e-12 already. Check that directly (a Gram
    // product, ~1/10 of a sweep) instead of running a verifying sweep.
    if (!__syncthreads_or(mid) && gram_orthogonal(U, ld, n, nrm, gram2, tid, nt)) {
      converged = true;
      break;
    }
  }
  if (tid == 0) {
    if (!converged) atomicCAS(&a.st->eig_fail, 0, bidx + 1);
    atomicAdd(&a.st->eig_sweeps, (unsigned long long)(sweep + 1));
#ifdef STROM_EIG_PROF
    if (bidx < 4096) g_eig_prof[bidx][7] = sweep + 1;
#endif
  }
  EIG_STAMP(3);
  // ---- 4. eigenpairs: lambda_j = ||u_j|| - s, v_j = u_j / ||u_j|| (u_j = (lambda_j + s) v_j) ---
  // Without GU: one thread per column (rows visited from a column-dependent start so a
  // half-warp's reads hit distinct banks); the columns stay unnormalised and wsc[j] =
  // 1/||u_j||^2 folds the normalisation into the reconstruction and the V store.
  __shared__ double wsc[256];     // [0, n): 1/||u_j||^2, [128, 128 + n): 1/||u_j||
  if (!GU) {
    for (int j = tid; j < n; j += nt) {
      const double *uj = U + j * ld;
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
      int i = j % n, c = 0;
      for (; c + 3 < n; c += 4) {
        const int i1 = i + 1 < n ? i + 1 : i + 1 - n;
        const int i2 = i1 + 1 < n ? i1 + 1 : i1 + 1 - n;
        const int i3 = i2 + 1 < n ? i2 + 1 : i2 + 1 - n;
        t0 += uj[i] * uj[i]; t1 += uj[i1] * uj[i1]; t2 += uj[i2] * uj[i2]; t3 += uj[i3] * uj[i3];
        i = i3 + 1 < n ? i3 + 1 : i3 + 1 - n;
      }
      for (; c < n; ++c) { t0 += uj[i] * uj[i]; i = i + 1 < n ? i + 1 : 0; }
      const double nn = (t0 + t1) + (t2 + t3);
      const double nr = sqrt(nn);
      lamv[j] = nr - s;
      wsc[j] = 1.0 / nn;
      wsc[128 + j] = 1.0 / nr;
    }
  } else {
    for (int j = warp; j < n; j += nwarps) {
      double *uj = U + j * ld;
      double nn = 0.0;
      for (int i = lane; i < n; i += 32) nn += uj[i] * uj[i];
      nn = warp_sum(nn);
      const double nr = sqrt(nn);
      if (lane == 0) lamv[j] = nr - s;
      if (proj || a.mode == 2) {     // mode 2 returns unit eigenvectors (strom.h)
        const double inv = 1.0 / nr;
        for (int i = lane; i < n; i += 32) uj[i] *= inv;
      }
    }
  }
  V = U;                          // eigenvectors now live in the U buffer
  __syncthreads();
  const double *lam = lamv;
  if (a.mode == 2) {
    double l1, l2;
    const int j = top2(lam, n, l1, l2);
    if (tid == 0) { a.lam12[2 * bidx] = l1; a.lam12[2 * bidx + 1] = l2; }
    const double inv = GU ? 1.0 : wsc[128 + j];
    const double sg = V[j * ld] < 0.0 ? -inv : inv;
    for (int i = tid; i < n; i += nt) a.vtop[a.toff[bidx] + i] = V[j * ld + i] * sg;
    return;
  }
  if (!proj) {
    // eigenvalue error floor for the certificate (PAPER.md:535-537 must never overstate
    // the bound): lambda_j = ||u_j|| - s carries an absolute error ~ n u (||Z||_F + s) =
    // 1.5 n u s (s = 2 ||Z||_F); the reported lambda_min is lowered by that margin.
    if (tid == 0) {
      double lm = lam[0];
      for (int k = 1; k < n; ++k) lm = fmin(lm, lam[k]);
      a.lam_min[bidx] = lm - 1.5 * n * 2.220446049250313e-16 * s;
    }
    return;
  }
  if (warp == 0) {                // the smaller eigen-set, ascending order, by ballots
    int npos = 0, nneg = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      const double l = k < n ? lam[k] : 0.0;
      npos += __popc(__ballot_sync(0xffffffffu, l > 0.0));
      nneg += __popc(__ballot_sync(0xffffffffu, l < 0.0));
    }
    const int use_pos = npos <= nneg;
    int cnt = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      const double l = k < n ? lam[k] : 0.0;
      const bool pick = use_pos ? (l > 0.0) : (l < 0.0);
      const unsigned b = __ballot_sync(0xffffffffu, pick);
      if (pick) sets[cnt + __popc(b & ((1u << lane) - 1u))] = k;
      cnt += __popc(b);
    }
    if (lane == 0) set_info = cnt * 2 + use_pos;
  }
  __syncthreads();
  const int cnt = set_info >> 1, use_pos = set_info & 1;
  const double is = 1.0 / sigma;
  if (!GU)                        // per selected eigenpair: lambda_k / ||u_k||^2
    for (int c = tid; c < cnt; c += nt) red[c] = lam[sets[c]] * wsc[sets[c]];
  __syncthreads();
  EIG_STAMP(4);
  // ---- 5. S = (Pi(X_b) - X_b)/sigma in svec ------------------------------------------
  // S entry (i <= j): from P_ij = sum_c w_c u_kc[i] u_kc[j] over the smaller eigen-set
  // (c ascending), either (P - X_b)/sigma (positive set) or -P/sigma (negative set).
  auto emit = [&](int i, int j, double acc) {
    const int e = j * (j + 1) / 2 + i;
    double sv;
    if (use_pos) {
      const double xb = Xb[e];
      sv = (acc - (i == j ? xb : xb * isq2)) * is;
    } else {
      sv = -acc * is;
    }
    a.S_out[off + e] = (i == j) ? sv : sv * 1.41421356237309504880;
  };
  const int nTr = (n + 3) >> 2;
  if (!GU && nTr * nTr <= nt) {
    // 4x4 register tiles over the full matrix (strided rows/columns as in the warm product)
    if (tid < nTr * nTr) {
      const int ti = tid % nTr, tj = tid / nTr;
      int ir[4], jc[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) { ir[r] = min(ti + nTr * r, n - 1); jc[r] = min(tj + nTr * r, n - 1); }
      double acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
      for (int c = 0; c < cnt; ++c) {
        const double *uk = V + sets[c] * ld;
        const double w = red[c];
        double x[4], z[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) { x[r] = w * uk[ir[r]]; z[r] = uk[jc[r]]; }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[r][q] += x[r] * z[q];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = ti + nTr * r, j = tj + nTr * q;
          if (i <= j && j < n) emit(i, j, acc[r][q]);
        }
    }
  } else {
    for (int e = tid; e < L; e += nt) {
      int i, j;
      svec_ij(e, i, j);
      double acc = 0.0;
      if (GU) {
        for (int c = 0; c < cnt; ++c) {
          const int k = sets[c];
          acc += lam[k] * V[k * ld + i] * V[k * ld + j];
        }
      } else {
        for (int c = 0; c < cnt; ++c) {
          const int k = sets[c];
          acc += red[c] * V[k * ld + i] * V[k * ld + j];
        }
      }
      emit(i, j, acc);
    }
  }
  // ---- 6. keep the eigenbasis for the next iteration -------------------------------
  EIG_STAMP(5);
  double *Vs = a.Vstore + a.voff[bidx];
  if (GU) {
    for (int e = tid; e < n * n; e += nt) Vs[e] = V[e];
  } else {
    for (int e = tid; e < n * n; e += nt) {
      const int j = e / n;
      Vs[e] = V[j * ld + e - j * n] * wsc[128 + j];
    }
  }
  __syncthreads();
  EIG_STAMP(6);
}

inline bool eig_global(int n) { return n > 112; }
inline int eig_G(int n);
inline size_t eig_smem_bytes(int n) {
  const int NP = n + (n & 1);
  const size_t mats = eig_global(n) ? 0 : 2 * (size_t)n * eig_ld(n, eig_G(n));
  return sizeof(double) * (mats + n + 8) + sizeof(unsigned short) * (size_t)(NP - 1) * (NP / 2) + 16;
}

// lanes per pair and launch shape for a block of order n
inline int eig_G(int n) {
  if (eig_global(n)) return 32;
  static int force = [] { const char *e = getenv("STROM_EIG_G"); return e ? atoi(e) : 0; }();
  if (force == 8 && n <= 112) return 8;
  if (force == 16 && n > 16) return 16;
  if (force == 32 && n > 16 && n <= 64) return 32;
  // 8 lanes per pair up to the shared-memory limit: at order 105 (cart-pole) one pass of
  // 14 warps per round instead of two passes with 16 lanes (K-EIG 479 -> 408 us)
  return n <= 16 ? 4 : (n <= 112 ? 8 : 16);
}
inline int eig_threads(int n) {
  const int H = (n + (n & 1)) / 2, G = eig_G(n), ppw = 32 / G;
  if (G == 32) return std::min(512, 32 * H);
  int warps = (H + ppw - 1) / ppw;
  int t = 32 * std::max(warps, 1);
  while (t < 512 && (int64_t)n * n > 16LL * t) t += 32;   // warm-start product capacity
  // n > 16: 16 warps. The rounds use ceil(H/4) of them (the rest only meet the barriers,
  // +1.5% per sweep); the gather, warm product, reconstruction and V traffic get twice the
  // threads (order 55: gather 19.7K -> 13.7K cycles, iteration 216.6 -> 207.7 us).
  static const int force_t = [] { const char *e = getenv("STROM_EIG_THREADS"); return e ? atoi(e) : 512; }();
  if (n > 16) t = std::max(t, std::max(256, force_t));
  return std::min(t, 512);
}

// ============================================================================
// K-EIG, cluster variant for orders 113..236 (car back-in / landing 190, flying robot
// 231). A 2-CTA cluster owns one block: CTA r holds rows
// [r*h, r*h + h) of U = X_b + sI (h = ceil(n/2)) for all n columns in its shared memory.
// Per round each CTA computes the partial dots u_p.u_q over its rows for every pair,
// publishes them in its shared memory, one cluster barrier, then both CTAs read both
// partials through DSMEM, sum them in a fixed order (identical in both CTAs), compute the
// same rotation and apply it to their own rows. Column norms are kept identical in both
// CTAs. Cold start (V = I) in this version; eigenvectors = normalised columns of U.
// ============================================================================
constexpr int kClusterEig = 2;

__host__ __device__ inline int eig_cluster_rows(int n) { return (n + kClusterEig - 1) / kClusterEig; }
inline bool eig_use_cluster(int n) { return n > 112 && n <= 236; }
// cluster size of the large-block K-EIG: 4 (k_eig_cl, default) or 2 (k_eig_cluster);
// STROM_EIG_CL=2 selects the 2-CTA kernel
inline int eig_cl_size() {
  static const int c = [] { const char *e = getenv("STROM_EIG_CL"); return e && atoi(e) == 2 ? 2 : 4; }();
  return c;
}
inline size_t eig_cluster_smem_bytes(int n) {
  const int NP = n + (n & 1), H = NP / 2, h = eig_cluster_rows(n);
  return sizeof(double) * ((size_t)h * n + n /*norms*/ + n /*lambda*/ + 2 * (size_t)H /*partials*/ + 16);
}

// G lanes per column pair, EPL >= h/G local rows per lane.
template <int G, int EPL>
__global__ void __cluster_dims__(kClusterEig, 1, 1) __launch_bounds__(512, 1) k_eig_cluster(EigArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  if (a.st->done) return;                     // uniform across the cluster
  extern __shared__ double sm[];
  __shared__ double red[4 * 32];
  __shared__ int sets[128];
  __shared__ int set_info;
  constexpr int PPW = 32 / G;
  const int crank = (int)cl.block_rank();
  const int bidx = a.blocks[blockIdx.x / kClusterEig];
  const int n = a.bn[bidx];
  const int NP = n + (n & 1), H = NP / 2;
  const int h = eig_cluster_rows(n);
  const int r0 = crank * h, nloc = min(h, n - r0);   // local rows [r0, r0 + nloc)
  const int64_t off = a.boff[bidx];
  const int L = n * (n + 1) / 2;
  double *U = sm;                                   // column j, local row i: U[j*h + i]
  double *nrm = sm + (size_t)h * n;                 // n
  double *lamv = nrm + n;                           // n
  double *part = lamv + n;                          // 2 x H (parity)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int grp = lane / G, sub = lane % G;
  const double sigma = a.st->sigma;
  const double isq2 = 0.70710678118654752440;
  const bool proj = (a.mode == 0);
  // ---- 1. gather X_b (each CTA half of the svec entries), Frobenius norm -------------
  double fro = gather_xb(a, off, L, crank * nt + tid, kClusterEig * nt, sigma, proj);
  {
    double v1[1] = {fro};
    block_sum<1>(v1, red);
    if (tid == 0) part[0] = v1[0];
  }
  cl.sync();                                        // Xb_out and both partial norms visible
  double s;
  {
    double tot = 0.0;
    for (int c = 0; c < kClusterEig; ++c) tot += cl.map_shared_rank(part, c)[0];
    s = 2.0 * sqrt(tot) + 1e-300;
  }
  cl.sync();                                        // partial slot reused below
  const double *Xb = a.Xb_out + off;
  // ---- 2. local rows of U = (X_b + sI) V, V = V_prev (warm) or I ------------------------
  const bool warm = proj && a.warm_enable && a.st->eig_warm_valid &&
                    (a.cold_every <= 0 || (a.st->iter % a.cold_every) != 0);
  if (warm) {
    // U[i, j] = sum_k A[i, k] V[k, j] + s V[i, j]; A from the L2-resident svec X_b, V_prev
    // column-major in global memory (column j is a warp-uniform broadcast stream)
    const double *Vp = a.Vstore + a.voff[bidx];
    for (int e = tid; e < nloc * n; e += nt) {
      const int j = e / nloc, il = e - j * nloc, i = r0 + il;
      const double *vj = Vp + (int64_t)j * n;
      double t0 = 0.0, t1 = 0.0;
      int k = 0;
      for (; k + 1 < n; k += 2) {
        const double a0 = Xb[svec_pos(i, k)], a1 = Xb[svec_pos(i, k + 1)];
        t0 += (i == k ? a0 : a0 * isq2) * vj[k];
        t1 += (i == k + 1 ? a1 : a1 * isq2) * vj[k + 1];
      }
      if (k < n) { const double a0 = Xb[svec_pos(i, k)]; t0 += (i == k ? a0 : a0 * isq2) * vj[k]; }
      U[j * h + il] = (t0 + t1) + s * vj[i];
    }
  } else {
    for (int e = tid; e < nloc * n; e += nt) {
      const int j = e / nloc, il = e - j * nloc, i = r0 + il;
      const double v = Xb[svec_pos(i, j)];
      U[j * h + il] = (i == j) ? v + s : v * isq2;
    }
  }
  __syncthreads();
  cl.sync();          // every CTA has read V_prev before anyone overwrites it (step 4)
  // ---- 3. sweeps ------------------------------------------------------------------------
  const double tol = fmax(a.tol, 4.0 * n * 2.220446049250313e-16);
  const double tol2 = tol * tol, quad2 = 1e-18;
  bool converged = false;
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    // exact column norms: partial over local rows, exchanged through DSMEM
    for (int j = warp; j < n; j += nwarps) {
      const double *uj = U + j * h;
      double t = 0.0;
      for (int i = lane; i < nloc; i += 32) t += uj[i] * uj[i];
      t = warp_sum(t);
      if (lane == 0) lamv[j] = t;
    }
    cl.sync();
    for (int j = tid; j < n; j += nt) {
      double t = 0.0;
      for (int c = 0; c < kClusterEig; ++c) t += cl.map_shared_rank(lamv, c)[j];
      nrm[j] = t;
    }
    cl.sync();                                      // lamv free again; nrm complete
    int rotated = 0, big = 0;
    for (int r = 0; r < NP - 1; ++r) {
      double *pr = part + (r & 1) * H;
      // phase A: partial dots over the local rows
      for (int P0 = warp * PPW; P0 < H; P0 += nwarps * PPW) {
        const int P = P0 + grp;
        int p = 0, q = 0;
        bool valid = P < H;
        if (valid) {
          p = rr_pos(P, r, NP - 1); q = rr_pos(NP - 1 - P, r, NP - 1);
          if (p > q) { const int t2 = p; p = q; q = t2; }
          valid = q < n;
        }
        double g0 = 0.0, g1 = 0.0;
        if (valid) {
          const double *up = U + p * h, *uq = U + q * h;
#pragma unroll
          for (int c = 0; c < EPL; ++c) {
            const int i = sub + G * c;
            if (i < nloc) { if (c & 1) g1 += up[i] * uq[i]; else g0 += up[i] * uq[i]; }
          }
        }
        const double ga = group_sum<G>(g0 + g1);
        if (valid && sub == 0) pr[P] = ga;
      }
      cl.sync();
      // phase B: identical rotations in both CTAs, applied to the local rows
      for (int P0 = warp * PPW; P0 < H; P0 += nwarps * PPW) {
        const int P = P0 + grp;
        if (P >= H) continue;
        int p = rr_pos(P, r, NP - 1), q = rr_pos(NP - 1 - P, r, NP - 1);
        if (p > q) { const int t2 = p; p = q; q = t2; }
        if (q >= n) continue;
        double ga = 0.0;
        for (int c = 0; c < kClusterEig; ++c) ga += cl.map_shared_rank(pr, c)[P];
        const double al = nrm[p], be = nrm[q];
        const double ab = al * be, g2a = ga * ga;
        if (ga != 0.0 && g2a > tol2 * ab) {
          rotated = 1;
          if (g2a > quad2 * ab) big = 1;
          double cs, sn;
          jacobi_cs(al, be, ga, cs, sn);
          double *up = U + p * h, *uq = U + q * h;
#pragma unroll
          for (int c = 0; c < EPL; ++c) {
            const int i = sub + G * c;
            if (i < nloc) {
              const double x = up[i], y = uq[i];
              up[i] = cs * x - sn * y; uq[i] = sn * x + cs * y;
            }
          }
          __syncwarp(G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G)));   // nrm reads before the write
          if (sub == 0) {
            const double c2 = cs * cs, s2 = sn * sn, csn = 2.0 * cs * sn * ga;
            nrm[p] = c2 * al - csn + s2 * be;
            nrm[q] = s2 * al + csn + c2 * be;
          }
        }
      }
      __syncthreads();
    }
    const int any_big = __syncthreads_or(big);
    const int any_rot = __syncthreads_or(rotated);
    if (!any_rot || !any_big) { converged = true; break; }
  }
  if (tid == 0 && crank == 0) {
    if (!converged) atomicCAS(&a.st->eig_fail, 0, bidx + 1);
    atomicAdd(&a.st->eig_sweeps, (unsigned long long)(sweep + 1));
  }
  // ---- 4. eigenpairs: exact norms (DSMEM), lambda = ||u|| - s, V = normalised U --------
  for (int j = warp; j < n; j += nwarps) {
    const double *uj = U + j * h;
    double t = 0.0;
    for (int i = lane; i < nloc; i += 32) t += uj[i] * uj[i];
    t = warp_sum(t);
    if (lane == 0) lamv[j] = t;
  }
  cl.sync();
  for (int j = tid; j < n; j += nt) {
    double t = 0.0;
    for (int c = 0; c < kClusterEig; ++c) t += cl.map_shared_rank(lamv, c)[j];
    nrm[j] = sqrt(t);                               // ||u_j||
  }
  cl.sync();
  for (int j = tid; j < n; j += nt) lamv[j] = nrm[j] - s;
  __syncthreads();
  const double *lam = lamv;
  if (a.mode == 2) {
    double l1, l2;
    const int j = top2(lam, n, l1, l2);
    if (tid == 0 && crank == 0) { a.lam12[2 * bidx] = l1; a.lam12[2 * bidx + 1] = l2; }
    const double v0 = cl.map_shared_rank(U, 0)[j * h];     // row 0 lives in CTA 0
    const double sg = v0 < 0.0 ? -1.0 / nrm[j] : 1.0 / nrm[j];
    for (int il = tid; il < nloc; il += nt) a.vtop[a.toff[bidx] + r0 + il] = U[j * h + il] * sg;
    cl.sync();                                      // CTA 0's shared memory read by CTA 1
    return;
  }
  if (!proj) {
    if (tid == 0 && crank == 0) {   // with the same error margin as k_eig
      double lm = lam[0];
      for (int k = 1; k < n; ++k) lm = fmin(lm, lam[k]);
      a.lam_min[bidx] = lm - 1.5 * n * 2.220446049250313e-16 * s;
    }
    return;
  }
  // normalised local rows -> global V (column-major n x n) for the reconstruction
  double *Vg = a.Vstore + a.voff[bidx];
  for (int e = tid; e < nloc * n; e += nt) {
    const int j = e / nloc, il = e - j * nloc;
    Vg[j * n + r0 + il] = U[j * h + il] / nrm[j];
  }
  if (tid == 0) {
    int npos = 0, nneg = 0;
    for (int k = 0; k < n; ++k) { if (lam[k] > 0.0) ++npos; else if (lam[k] < 0.0) ++nneg; }
    const int use_pos = npos <= nneg;
    int cnt = 0;
    for (int k = 0; k < n; ++k)
      if (use_pos ? (lam[k] > 0.0) : (lam[k] < 0.0)) sets[cnt++] = k;
    set_info = cnt * 2 + use_pos;
  }
  __threadfence();
  cl.sync();                                        // V rows of both CTAs visible in global
  const int cnt = set_info >> 1, use_pos = set_info & 1;
  const double is = 1.0 / sigma;
  for (int e = crank * nt + tid; e < L; e += kClusterEig * nt) {
    int j = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (j * (j + 1) / 2 > e) --j;
    while ((j + 1) * (j + 2) / 2 <= e) ++j;
    const int i = e - j * (j + 1) / 2;
    double acc = 0.0;
    for (int c = 0; c < cnt; ++c) {
      const int k = sets[c];
      acc += lam[k] * Vg[k * n + i] * Vg[k * n + j];
    }
    double sv;
    if (use_pos) {
      const double xb = Xb[e];
      sv = (acc - (i == j ? xb : xb * isq2)) * is;
    } else {
      sv = -acc * is;
    }
    a.S_out[off + e] = (i == j) ? sv : sv * 1.41421356237309504880;
  }
}

// ============================================================================
// K-EIG, CL-CTA cluster variant with register-resident pairs (orders 113..236; car
// back-in / landing 190, flying robot 231). CTA r of the cluster holds
// rows [r h, r h + h) of U = (X_b + sI) V (h = ceil(n / CL)). One round: G lanes own a
// column pair for ALL pairs at once (CL = 4: 48-58 local rows, G = 4 -> 128 pairs per
// pass >= n/2), load its local rows into registers, form the partial dot, publish it; one
// cluster barrier; every CTA sums the CL partials in rank order (identical rotations in
// all CTAs), rotates the registers and stores them back; one CTA barrier. U is read and
// written once per round (the 2-CTA kernel above reads it twice and runs 3 passes).
// ============================================================================
__host__ __device__ inline int eig_cl_rows(int n, int CL) { return (n + CL - 1) / CL; }
// column stride (doubles) of the local rows: >= h and == 4 (mod 16), so the 4-double row
// segments that the 8 lane groups of a warp read from (mostly consecutive) columns start
// at banks 0, 8, 16, 24 in turn: two wavefronts per load instead of eight (h = 48)
__host__ __device__ inline int eig_cl_ld(int h) { return (h + 11) / 16 * 16 + 4; }
inline size_t eig_cl_smem_bytes(int n, int CL) {
  const int NP = n + (n & 1), H = NP / 2, ld = eig_cl_ld(eig_cl_rows(n, CL));
  return sizeof(double) * ((size_t)ld * n + n /*norms*/ + n /*lambda*/ + 2 * (size_t)H /*partials*/ + 16);
}

template <int CL, int G, int EPL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(512, 1) k_eig_cl(EigArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  if (a.st->done) return;                     // uniform across the cluster
  extern __shared__ double sm[];
  __shared__ double red[4 * 32];
  __shared__ int sets[128];
  __shared__ int set_info;
  constexpr int PPW = 32 / G;
  const int crank = (int)cl.block_rank();
  const int bidx = a.blocks[blockIdx.x / CL];
  const int n = a.bn[bidx];
  const int NP = n + (n & 1), H = NP / 2;
  const int h = eig_cl_rows(n, CL);
  const int r0 = crank * h, nloc = max(0, min(h, n - r0));   // local rows [r0, r0 + nloc)
  const int64_t off = a.boff[bidx];
  const int L = n * (n + 1) / 2;
  const int ldc = eig_cl_ld(h);
  double *U = sm;                                   // column j, local row i: U[j*ldc + i]
  double *nrm = sm + (size_t)ldc * n;               // n
  double *lamv = nrm + n;                           // n
  double *part = lamv + n;                          // 2 x H (parity)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  const int grp = lane / G, sub = lane % G;
  const double sigma = a.st->sigma;
  const double isq2 = 0.70710678118654752440;
  const bool proj = (a.mode == 0);
  // ---- 1. gather X_b (each CTA 1/CL of the svec entries), Frobenius norm ---------------
  double fro = gather_xb(a, off, L, crank * nt + tid, CL * nt, sigma, proj);
  {
    double v1[1] = {fro};
    block_sum<1>(v1, red);
    if (tid == 0) part[0] = v1[0];
  }
  cl.sync();                                        // Xb_out and every partial norm visible
  double s;
  {
    double tot = 0.0;
    for (int c = 0; c < CL; ++c) tot += cl.map_shared_rank(part, c)[0];
    s = 2.0 * sqrt(tot) + 1e-300;
  }
  cl.sync();                                        // partial slot reused below
  const double *Xb = a.Xb_out + off;
  // ---- 2. local rows of U = (X_b + sI) V, V = V_prev (warm) or I ------------------------
  const bool warm = proj && a.warm_enable && a.st->eig_warm_valid &&
                    (a.cold_every <= 0 || (a.st->iter % a.cold_every) != 0);
  if (warm) {
    const double *Vp = a.Vstore + a.voff[bidx];
    for (int e = tid; e < nloc * n; e += nt) {
      const int j = e / nloc, il = e - j * nloc, i = r0 + il;
      const double *vj = Vp + (int64_t)j * n;
      double t0 = 0.0, t1 = 0.0;
      int k = 0;
      for (; k + 1 < n; k += 2) {
        const double a0 = Xb[svec_pos(i, k)], a1 = Xb[svec_pos(i, k + 1)];
        t0 += (i == k ? a0 : a0 * isq2) * vj[k];
        t1 += (i == k + 1 ? a1 : a1 * isq2) * vj[k + 1];
      }
      if (k < n) { const double a0 = Xb[svec_pos(i, k)]; t0 += (i == k ? a0 : a0 * isq2) * vj[k]; }
      U[j * ldc + il] = (t0 + t1) + s * vj[i];
    }
  } else {
    for (int e = tid; e < nloc * n; e += nt) {
      const int j = e / nloc, il = e - j * nloc, i = r0 + il;
      const double v = Xb[svec_pos(i, j)];
      U[j * ldc + il] = (i == j) ? v + s : v * isq2;
    }
  }
  __syncthreads();
  cl.sync();          // every CTA has read V_prev before anyone overwrites it (step 4)
  // ---- 3. sweeps --------------------------------------------------------------------------
  const double tol = fmax(a.tol, 4.0 * n * 2.220446049250313e-16);
  const double tol2 = tol * tol, quad2 = 1e-18;
  bool converged = false;
  int sweep = 0;
  const int P = warp * PPW + grp;                   // this lane group's pair slot (one pass)
  for (; sweep < a.max_sweeps; ++sweep) {
    for (int j = warp; j < n; j += nwarps) {        // exact column norms (DSMEM sum)
      const double *uj = U + j * ldc;
      double t = 0.0;
      for (int i = lane; i < nloc; i += 32) t += uj[i] * uj[i];
      t = warp_sum(t);
      if (lane == 0) lamv[j] = t;
    }
    cl.sync();
    for (int j = tid; j < n; j += nt) {
      double t = 0.0;
      for (int c = 0; c < CL; ++c) t += cl.map_shared_rank(lamv, c)[j];
      nrm[j] = t;
    }
    cl.sync();                                      // lamv free again; nrm complete
    int rotated = 0, big = 0;
    for (int r = 0; r < NP - 1; ++r) {
      double *pr = part + (r & 1) * H;
      int p = 0, q = 0;
      bool valid = P < H;
      if (valid) {
        p = rr_pos(P, r, NP - 1); q = rr_pos(NP - 1 - P, r, NP - 1);
        if (p > q) { const int t2 = p; p = q; q = t2; }
        valid = q < n;
      }
      double xp[EPL], xq[EPL];
      double g0 = 0.0, g1 = 0.0;
      double *up = U + p * ldc, *uq = U + q * ldc;
#pragma unroll
      for (int c = 0; c < EPL; ++c) {
        const int i = sub + G * c;
        const bool ok = valid && i < nloc;
        xp[c] = ok ? up[i] : 0.0;
        xq[c] = ok ? uq[i] : 0.0;
        if (c & 1) g1 += xp[c] * xq[c]; else g0 += xp[c] * xq[c];
      }
      const double gl = group_sum<G>(g0 + g1);
      if (valid && sub == 0) pr[P] = gl;
      cl.sync();                                    // every CTA's partial dot visible
      if (valid) {
        double ga = 0.0;
        for (int c = 0; c < CL; ++c) ga += cl.map_shared_rank(pr, c)[P];
        const double al = nrm[p], be = nrm[q];
        const double ab = al * be, g2a = ga * ga;
        if (ga != 0.0 && g2a > tol2 * ab) {
          rotated = 1;
          if (g2a > quad2 * ab) big = 1;
          double cs, sn;
          jacobi_cs(al, be, ga, cs, sn);
#pragma unroll
          for (int c = 0; c < EPL; ++c) {
            const int i = sub + G * c;
            if (i < nloc) { up[i] = cs * xp[c] - sn * xq[c]; uq[i] = sn * xp[c] + cs * xq[c]; }
          }
          __syncwarp(G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G)));   // nrm reads before the write
          if (sub == 0) {
            const double c2 = cs * cs, s2 = sn * sn, csn = 2.0 * cs * sn * ga;
            nrm[p] = c2 * al - csn + s2 * be;
            nrm[q] = s2 * al + csn + c2 * be;
          }
        }
      }
      __syncthreads();                              // rotated columns visible to the next round
    }
    const int any_big = __syncthreads_or(big);
    const int any_rot = __syncthreads_or(rotated);
    if (!any_rot || !any_big) { converged = true; break; }
  }
  if (tid == 0 && crank == 0) {
    if (!converged) atomicCAS(&a.st->eig_fail, 0, bidx + 1);
    atomicAdd(&a.st->eig_sweeps, (unsigned long long)(sweep + 1));
  }
  // ---- 4. eigenpairs: exact norms (DSMEM), lambda = ||u|| - s, V = normalised U --------
  for (int j = warp; j < n; j += nwarps) {
    const double *uj = U + j * ldc;
    double t = 0.0;
    for (int i = lane; i < nloc; i += 32) t += uj[i] * uj[i];
    t = warp_sum(t);
    if (lane == 0) lamv[j] = t;
  }
  cl.sync();
  for (int j = tid; j < n; j += nt) {
    double t = 0.0;
    for (int c = 0; c < CL; ++c) t += cl.map_shared_rank(lamv, c)[j];
    nrm[j] = sqrt(t);                               // ||u_j||
  }
  cl.sync();
  for (int j = tid; j < n; j += nt) lamv[j] = nrm[j] - s;
  __syncthreads();
  const double *lam = lamv;
  if (a.mode == 2) {
    double l1, l2;
    const int j = top2(lam, n, l1, l2);
    if (tid == 0 && crank == 0) { a.lam12[2 * bidx] = l1; a.lam12[2 * bidx + 1] = l2; }
    const double v0 = cl.map_shared_rank(U, 0)[j * ldc];     // row 0 lives in CTA 0
    const double sg = v0 < 0.0 ? -1.0 / nrm[j] : 1.0 / nrm[j];
    for (int il = tid; il < nloc; il += nt) a.vtop[a.toff[bidx] + r0 + il] = U[j * ldc + il] * sg;
    cl.sync();                                      // CTA 0's shared memory read by the others
    return;
  }
  if (!proj) {
    if (tid == 0 && crank == 0) {   // with the same error margin as k_eig
      double lm = lam[0];
      for (int k = 1; k < n; ++k) lm = fmin(lm, lam[k]);
      a.lam_min[bidx] = lm - 1.5 * n * 2.220446049250313e-16 * s;
    }
    return;
  }
  // normalised local rows -> global V (column-major n x n) for the reconstruction
  double *Vg = a.Vstore + a.voff[bidx];
  for (int e = tid; e < nloc * n; e += nt) {
    const int j = e / nloc, il = e - j * nloc;
    Vg[j * n + r0 + il] = U[j * ldc + il] / nrm[j];
  }
  if (warp == 0) {                // the smaller eigen-set, ascending order, by ballots
    int npos = 0, nneg = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      const double l = k < n ? lam[k] : 0.0;
      npos += __popc(__ballot_sync(0xffffffffu, l > 0.0));
      nneg += __popc(__ballot_sync(0xffffffffu, l < 0.0));
    }
    const int use_pos = npos <= nneg;
    int cnt = 0;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int k = k0 + lane;
      const double l = k < n ? lam[k] : 0.0;
      const bool pick = use_pos ? (l > 0.0) : (l < 0.0);
      const unsigned b = __ballot_sync(0xffffffffu, pick);
      if (pick) sets[cnt + __popc(b & ((1u << lane) - 1u))] = k;
      cnt += __popc(b);
    }
    if (lane == 0) set_info = cnt * 2 + use_pos;
  }
  __threadfence();
  cl.sync();                                        // V rows of every CTA visible in global
  const int cnt = set_info >> 1, use_pos = set_info & 1;
  const double is = 1.0 / sigma;
  for (int e = crank * nt + tid; e < L; e += CL * nt) {
    int i, j;
    svec_ij(e, i, j);
    double acc = 0.0;
    for (int c = 0; c < cnt; ++c) {
      const int k = sets[c];
      acc += lam[k] * Vg[k * n + i] * Vg[k * n + j];
    }
    double sv;
    if (use_pos) {
      const double xb = Xb[e];
      sv = (acc - (i == j ? xb : xb * isq2)) * is;
    } else {
      sv = -acc * is;
    }
    a.S_out[off + e] = (i == j) ? sv : sv * 1.41421356237309504880;
  }
}
