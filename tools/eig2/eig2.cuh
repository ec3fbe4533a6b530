// MEASURED AND REJECTED: two-sided parallel Jacobi K-EIG variant, kept as a
// record with its numbers (profiles/r02b/README.md); not part of the build. It was wired into
// engine.cu launch_eig for mode 0, orders 6..64, and passed the projection / 50-iteration parity tests.

// K-EIG2: batched PSD-cone projection (Step 2 of Algorithm 1; projection
// Pi(X) = Q max(0, W) Q^T) by a two-sided parallel Jacobi, for blocks of
// order <= 64 (pendulum 55/10, cart-pole 14, car back-in / landing 19, flying robot 21).
// Included by engine.cu after eig.cuh (shares EigArgs, the gather and the rotation helpers).
//
// One CTA per block X_b, fp64 throughout:
//   1. gather X_b = X + sigma (A* y - C) from svec (A* fused), ||X_b||_F;
//   2. warm start B = V^T X_b V with V the block's eigenbasis of the previous iteration
//      (two 4x4-register-tile products; every 8th iteration V is first re-orthogonalised by
//      one Newton-Schulz step V <- 1.5 V - 0.5 V (V^T V), so the rounding of the accumulated
//      rotations cannot build up); cold: B = X_b, V = I;
//   3. rounds of the round-robin (circle) ordering: in one round every index pair (p, q) of
//      the round is rotated at once, B <- J^T B J, V <- V J (J the product of the round's
//      disjoint Givens rotations). The state of B is symmetric, stored full in shared
//      memory; thread t owns the 2x2 block (P, Q) of pair slots P <= Q and applies
//      J_P^T [.] J_Q to it. The rotation of a pair of the NEXT round is computed by the
//      owner of the block that holds its off-diagonal entry (it has the entry's new value
//      and the pair's new diagonal from the two current rotations), so a round needs ONE
//      CTA barrier -- __syncthreads_or of "some off-diagonal |b_ij| > thr", which is also
//      the exit test (every off-diagonal entry is rewritten, and tested, every round);
//   4. lambda_j = b_jj, v_j = V e_j (orthonormal); S = (Pi(X_b) - X_b)/sigma from the
//      smaller eigen-set (Moreau), as in k_eig; V kept for the next iteration.
// Versus the one-sided k_eig: a round has no column dot product (no shuffle reduction:
// the pair's entries are read directly), and the rotation of the next round is computed
// while the current one is applied, so the dependent chain per round is one rotation plus
// one 2x2 update plus one barrier.

struct Rot2 { double c, s, a, d; };   // rotation (c, s) of a pair and its new diagonal (a, d)

// Givens rotation zeroing b_pq of [[a, g], [g, d]] (same angle as jacobi_cs: tan(2 theta) =
// 2g / (d - a), |theta| <= pi/4), identity when |g| <= thr. Branch-free (the lanes of a warp
// take the same path): MUFU rsqrt / rcp refined by Newton steps, (c, s) orthogonal to fp64
// precision. New diagonal by the accurate update a - t g, d + t g (t = tan theta).
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
  Rot2 R;
  R.c = on ? cs : 1.0; R.s = on ? cs * t : 0.0;
  R.a = fma(-t, g, a); R.d = fma(t, g, d);
  return R;
}

// dst = alpha op(A) Bm + beta Cm for n x n column-major operands (stride ld), op(A) = A^T
// (TA) or A; 4x4 register tiles (ceil(n/4)^2 <= blockDim.x), every read before one CTA
// barrier, then the write: dst may alias any operand. k-sums in k order.
template <bool TA>
__device__ __forceinline__ void mm_tiles(const double *Am, const double *Bm, double *dst, int n, int ld,
                                         double alpha, double beta, const double *Cm) {
  const int tid = threadIdx.x, nT = (n + 3) >> 2;
  const bool act = tid < nT * nT;
  const int ti = act ? tid % nT : 0, tj = act ? tid / nT : 0;
  int ir[4], jc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) { ir[r] = min(ti + nT * r, n - 1); jc[r] = min(tj + nT * r, n - 1); }
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  if (act) {
#pragma unroll 2
    for (int k = 0; k < n; ++k) {
      double x[4], z[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        x[r] = TA ? Am[ir[r] * ld + k] : Am[k * ld + ir[r]];
        z[r] = Bm[jc[r] * ld + k];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(x[r], z[c], acc[r][c]);
    }
  }
  double cv[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) cv[r][c] = (act && beta != 0.0) ? Cm[jc[c] * ld + ir[r]] : 0.0;
  __syncthreads();
  if (act) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = ti + nT * r, j = tj + nT * c;
        if (i < n && j < n) dst[j * ld + i] = fma(alpha, acc[r][c], beta * cv[r][c]);
      }
  }
}

__host__ __device__ inline int eig2_ld(int NP) { return NP + 2; }   // even (16 B rows), != 0 mod 16
// K-EIG2 for the projection of blocks of (even-padded) order <= 64; STROM_EIG2=0 selects
// the one-sided k_eig instead
inline bool eig2_use(int np) {
  static const int on = [] { const char *e = getenv("STROM_EIG2"); return e ? atoi(e) : 1; }();
  return on && np >= 6 && np <= 64;
}
inline size_t eig2_smem_bytes(int np) {
  const int H = np / 2, ld = eig2_ld(np);
  return sizeof(double) * (3 * (size_t)np * ld + np + 8) + sizeof(Rot2) * 2 * H +
         sizeof(unsigned short) * (size_t)(np - 1) * H + 16;
}
inline int eig2_threads(int np) {
  const int H = np / 2, nb = H * (H + 1) / 2, nT = (np + 3) / 4;
  int t = std::max(nb, nT * nT);
  t = std::max(t, H * H / 2);
  t = (t + 31) / 32 * 32;
  return std::min(512, std::max(64, t));
}

__global__ void __launch_bounds__(512, 1) k_eig2(EigArgs a) {
  pdl_trigger();
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[4 * 32];
  __shared__ int sets[128];
  __shared__ int set_info;
  const int bidx = a.blocks[blockIdx.x];
  const int n = a.bn[bidx];
  const int NP = n + (n & 1), H = NP / 2, M = NP - 1;
  const int64_t off = a.boff[bidx];
  const int L = n * (n + 1) / 2;
  const int ld = eig2_ld(NP);
  double *Bm = sm;                         // X_b, then T = X_b V, then B (NP x ld)
  double *V = sm + NP * ld;                // eigenbasis (column j = v_j)
  double *W = sm + 2 * NP * ld;            // scratch (V^T V)
  double *lamv = sm + 3 * NP * ld;
  Rot2 *rec = (Rot2 *)(lamv + NP + 8);     // [2][H]: rotations of the current / next round
  unsigned short *sched = (unsigned short *)(rec + 2 * H);   // (p | q << 8) per (round, slot)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const double isq2 = 0.70710678118654752440;
  // slot S of round r pairs the elements at circle positions S ("first") and M - S
  // ("second"); roles by position, not by index order
  EIG_STAMP(0);
  for (int e = tid; e < M * H; e += nt) {
    const int r = e / H, P = e - r * H;
    sched[e] = (unsigned short)(rr_pos(P, r, M) | (rr_pos(M - P, r, M) << 8));
  }
  // This thread's (at most two) 2x2 blocks (P <= Q) and V blocks (row pair I, slot Q), and
  // the static producer roles. The elements at positions j of round r move to position j-1
  // in round r+1 (position 1 -> M, 0 fixed), so the pair of next-round slot P' is made of
  // the current positions P'+1 and M-P'+1: slot P' (1 <= P' <= H-2) comes from block
  // (P'-1, P'+1) as (first of P'+1, second of P'-1) = entry n10; slot 0 from block (0, 1)
  // as (first of 0, first of 1) = n00; slot H-1 from block (H-2, H-1) as (second of H-1,
  // second of H-2) = n11. H >= 3 (order >= 5): every block produces at most one pair.
  const int NB = H * (H + 1) / 2, nV = H * H;
  int bP[2], bQ[2], bprod[2], vI[2], vQ[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int t = tid + k * nt;
    bP[k] = -1; bQ[k] = 0; bprod[k] = 0;
    if (t < NB) {
      int P = 0, rem = t;
      while (rem >= H - P) { rem -= H - P; ++P; }
      const int Q = P + rem;
      bP[k] = P; bQ[k] = Q;
      if (P == 0 && Q == 1) bprod[k] |= 1;                     // n00 -> slot 0
      if (P == H - 2 && Q == H - 1) bprod[k] |= 2;             // n11 -> slot H-1
      if (Q == P + 2) bprod[k] |= 4;                           // n10 -> slot P+1
    }
    vI[k] = -1; vQ[k] = 0;
    const int tv = tid + k * nt;
    if (tv < nV) { vI[k] = tv % H; vQ[k] = tv / H; }
  }
  pdl_wait();
  if (a.st->done) return;
  const double sigma = a.st->sigma;
  const bool warm = a.warm_enable && a.st->eig_warm_valid &&
                    (a.cold_every <= 0 || (a.st->iter % a.cold_every) != 0);
  const bool reorth = warm && (a.st->iter & 7) == 0;
  // ---- 1. gather X_b ---------------------------------------------------------------
  constexpr int KE = 12;
  const bool fast = (int64_t)(a.Atp[off + L] - a.Atp[off]) <= 3LL * NP * ld && L <= KE * nt;
  double xv[KE];
  double fro = fast ? gather_xb_smem<KE>(a, off, L, sm, xv, sigma, true)
                    : gather_xb(a, off, L, tid, nt, sigma, true);
  {
    double v1[1] = {fro};
    block_sum<1>(v1, red);
    if (tid == 0) red[127] = sqrt(v1[0]);
    __syncthreads();
  }
  const double nrmF = red[127];
  EIG_STAMP(1);
  const double *Xb = a.Xb_out + off;
  // ---- 2. B (X_b staged symmetric, padding rows/columns zero), V -------------------------
  for (int e = tid; e < NP * ld; e += nt) { const int j = e / ld, i = e - j * ld; if (i >= n || j >= n) Bm[e] = 0.0; }
  if (fast) {
#pragma unroll
    for (int k = 0; k < KE; ++k) {
      const int e = tid + k * nt;
      if (e < L) {
        int i, j;
        svec_ij(e, i, j);
        if (i == j) Bm[j * ld + i] = xv[k];
        else { const double v = xv[k] * isq2; Bm[j * ld + i] = v; Bm[i * ld + j] = v; }
      }
    }
  } else {
    for (int e = tid; e < n * n; e += nt) {
      const int j = e / n, i = e - j * n;
      const double v = Xb[svec_pos(i, j)];
      Bm[j * ld + i] = (i == j) ? v : v * isq2;
    }
  }
  if (warm) {
    const double *Vp = a.Vstore + a.voff[bidx];
    for (int e = tid; e < NP * ld; e += nt) {
      const int j = e / ld, i = e - j * ld;
      V[e] = (i < n && j < n) ? Vp[j * n + i] : 0.0;
    }
    __syncthreads();
    if (reorth) {
      mm_tiles<true>(V, V, W, n, ld, 1.0, 0.0, nullptr);          // W = V^T V
      __syncthreads();
      mm_tiles<false>(V, W, V, n, ld, -0.5, 1.5, V);              // V = 1.5 V - 0.5 V W
      __syncthreads();
    }
    mm_tiles<false>(Bm, V, Bm, n, ld, 1.0, 0.0, nullptr);         // T = X_b V
    __syncthreads();
    mm_tiles<true>(V, Bm, Bm, n, ld, 1.0, 0.0, nullptr);          // B = V^T T
  } else {
    for (int e = tid; e < NP * ld; e += nt) {
      const int j = e / ld, i = e - j * ld;
      V[e] = (i == j && i < n) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  EIG_STAMP(2);
  // ---- 3. Jacobi rounds -----------------------------------------------------------------
  const double thr = fmax(a.tol, 1e-16) * nrmF, thr2 = thr * thr;
  int big = 0;
  for (int e = tid; e < n * ld; e += nt) {
    const int j = e / ld, i = e - j * ld;
    if (i < n && i != j && fabs(Bm[e]) > thr) big = 1;
  }
  for (int P = tid; P < H; P += nt) {
    const unsigned fs = sched[P];
    const int f = fs & 0xff, sc = fs >> 8;
    rec[P] = rot2(Bm[f * ld + f], Bm[sc * ld + sc], Bm[sc * ld + f], thr);
  }
  big = __syncthreads_or(big);
  const int maxr = a.max_sweeps * M;
  int rounds = 0, r = 0;
#ifdef STROM_EIG_PROF
  long long tp[4] = {0, 0, 0, 0}, tq = clock64();
#define EIG2_T(k) do { if (tid == 2) { const long long tn = clock64(); tp[k] += tn - tq; tq = tn; } } while (0)
#else
#define EIG2_T(k) do { } while (0)
#endif
  while (big && rounds < maxr) {
    const Rot2 *rc = rec + (rounds & 1) * H;
    Rot2 *rn = rec + ((rounds + 1) & 1) * H;
    const unsigned short *sr = sched + r * H;
    int mybig = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (bP[k] < 0) continue;
      const int P = bP[k], Q = bQ[k];
      const unsigned fs1 = sr[P];
      const int f1 = fs1 & 0xff, s1 = fs1 >> 8;
      const Rot2 R1 = rc[P];
      if (P == Q) {
        Bm[f1 * ld + f1] = R1.a; Bm[s1 * ld + s1] = R1.d;
        Bm[s1 * ld + f1] = 0.0; Bm[f1 * ld + s1] = 0.0;
        continue;
      }
      const unsigned fs2 = sr[Q];
      const int f2 = fs2 & 0xff, s2 = fs2 >> 8;
      const Rot2 R2 = rc[Q];
      const double b00 = Bm[f2 * ld + f1], b01 = Bm[s2 * ld + f1];
      const double b10 = Bm[f2 * ld + s1], b11 = Bm[s2 * ld + s1];
      // right: [b] J_Q, then left: J_P^T [m]
      const double m00 = R2.c * b00 - R2.s * b01, m01 = R2.s * b00 + R2.c * b01;
      const double m10 = R2.c * b10 - R2.s * b11, m11 = R2.s * b10 + R2.c * b11;
      const double n00 = R1.c * m00 - R1.s * m10, n10 = R1.s * m00 + R1.c * m10;
      const double n01 = R1.c * m01 - R1.s * m11, n11 = R1.s * m01 + R1.c * m11;
      EIG2_T(0);
      // producer (H >= 3: at most one next-round pair per block; one rot2 per warp)
      const int pr = bprod[k];
      if (pr) {
        const bool sf = pr & 4, ff = pr & 1;
        const double pa = sf ? R2.a : ff ? R1.a : R2.d;      // (first of Q, second of P) |
        const double pd = sf ? R1.d : ff ? R2.a : R1.d;      // (first of 0, first of 1) |
        const double pg = sf ? n10 : ff ? n00 : n11;         // (second of H-1, second of H-2)
        rn[sf ? P + 1 : ff ? 0 : H - 1] = rot2(pa, pd, pg, thr);
      }
      EIG2_T(1);
      Bm[f2 * ld + f1] = n00; Bm[f1 * ld + f2] = n00;
      Bm[s2 * ld + f1] = n01; Bm[f1 * ld + s2] = n01;
      Bm[f2 * ld + s1] = n10; Bm[s1 * ld + f2] = n10;
      Bm[s2 * ld + s1] = n11; Bm[s1 * ld + s2] = n11;
      if (fma(n00, n00, fma(n01, n01, fma(n10, n10, n11 * n11))) > thr2) mybig = 1;
    }
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
    EIG2_T(2);
    big = __syncthreads_or(mybig);
    if (big) EIG2_T(3);
    ++rounds;
    r = (r + 1 == M) ? 0 : r + 1;
  }
  if (tid == 0) {
    if (big) atomicCAS(&a.st->eig_fail, 0, bidx + 1);
    atomicAdd(&a.st->eig_sweeps, (unsigned long long)((rounds + M - 1) / M));
  }
#ifdef STROM_EIG_PROF
  if (tid == 2 && bidx < 4096) {
    g_eig_prof[bidx][7] = rounds;     // rounds, not sweeps
    for (int k = 0; k < 4; ++k) g_eig_prof[bidx][12 + k] = tp[k];
  }
#endif
  EIG_STAMP(3);
  // ---- 4. eigenpairs, the smaller eigen-set -------------------------------------------
  for (int j = tid; j < n; j += nt) lamv[j] = Bm[j * ld + j];
  __syncthreads();
  const double *lam = lamv;
  if (warp == 0) {
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
  for (int c = tid; c < cnt; c += nt) red[c] = lam[sets[c]];
  __syncthreads();
  EIG_STAMP(4);
  // ---- 5. S = (Pi(X_b) - X_b)/sigma in svec: P_ij = sum_c lambda_c v_c[i] v_c[j] ----------
  const int nTr = (n + 3) >> 2;
  if (tid < nTr * nTr) {
    const int ti = tid % nTr, tj = tid / nTr;
    int ir[4], jc[4];
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2) { ir[r2] = min(ti + nTr * r2, n - 1); jc[r2] = min(tj + nTr * r2, n - 1); }
    double acc[4][4];
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r2][c] = 0.0;
    for (int c = 0; c < cnt; ++c) {
      const double *uk = V + sets[c] * ld;
      const double w = red[c];
      double x[4], z[4];
#pragma unroll
      for (int r2 = 0; r2 < 4; ++r2) { x[r2] = w * uk[ir[r2]]; z[r2] = uk[jc[r2]]; }
#pragma unroll
      for (int r2 = 0; r2 < 4; ++r2)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[r2][q] += x[r2] * z[q];
    }
#pragma unroll
    for (int r2 = 0; r2 < 4; ++r2)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = ti + nTr * r2, j = tj + nTr * q;
        if (i <= j && j < n) {
          const int e = j * (j + 1) / 2 + i;
          double sv;
          if (use_pos) {
            const double xb = Xb[e];
            sv = (acc[r2][q] - (i == j ? xb : xb * isq2)) * is;
          } else {
            sv = -acc[r2][q] * is;
          }
          a.S_out[off + e] = (i == j) ? sv : sv * 1.41421356237309504880;
        }
      }
  }
  EIG_STAMP(5);
  // ---- 6. keep the eigenbasis ----------------------------------------------------------
  double *Vs = a.Vstore + a.voff[bidx];
  for (int e = tid; e < n * n; e += nt) {
    const int j = e / n;
    Vs[e] = V[j * ld + e - j * n];
  }
  __syncthreads();
  EIG_STAMP(6);
}
