// Horizon partition of the chain across ranks (PAPER.md:606 distributes
// the moment blocks over GPUs): rank q owns the stages [cut[q], cut[q+1]), i.e. their PSD
// blocks, leaf rows, interior rows R_k and the separators between two of its stages. The
// separator S_j with j = cut[q+1] - 1 couples rank q and q+1: it is a *boundary*
// separator, and the only coupling left after each rank eliminates its own rows.
//
// With the separators ordered [internal of rank 0] ... [internal of rank R-1] [boundary],
// the separator Schur complement T of eps I + AA* is
//     T = [ blockdiag_q T_II^q   T_IB ]      T_IB^q couples rank q's internal
//         [ T_BI                 T_BB ]      separators to its two adjacent boundaries,
// and T y = u is solved by
//     u~_B = u_B - sum_q W^qT u_I^q,  W^q = (T_II^q)^{-1} T_IB^q          (one allreduce)
//     y_B  = T~^{-1} u~_B,            T~  = T_BB - sum_q T_BI^q W^q       (replicated)
//     y_I^q = (T_II^q)^{-1} u_I^q - W^q y_B                               (local)
// Every term of u~_B is a sum of rank-local partials (boundary rows touch the blocks of
// two ranks), so ONE sum-allreduce of |B| doubles per solve is the whole exchange.
//
// This file holds the plan (which rows each rank owns) and a host execution of the
// partitioned solve (setup factors with the dense host routines) used by CPU tests and
// the world-size-2 gloo test; the device path (engine.cu) computes the same factors with
// cuSOLVER at setup and runs the phases in sm_100a kernels.
#include <algorithm>
#include <cmath>

#include "host.h"

namespace strom {

strom_status make_plan(const Sdp &s, const Factor &f, int R, int r, PartPlan &p) {
  const int P = f.P;
  if (R < 1 || r < 0 || r >= R || R > P) {
    set_error("partition: need 1 <= nranks <= number of stages and 0 <= rank < nranks");
    return STROM_EINVAL;
  }
  p = PartPlan();
  p.R = R; p.r = r;
  // contiguous stage ranges balanced by the projection work sum n_beta^3 (+1 per stage)
  std::vector<double> cost(P, 1.0);
  for (int k = 0; k < s.nblocks; ++k) cost[s.bstage[k]] += (double)s.bn[k] * s.bn[k] * s.bn[k];
  double tot = 0.0;
  for (double c : cost) tot += c;
  p.cut.assign(R + 1, P);
  p.cut[0] = 0;
  double acc = 0.0;
  int q = 1;
  for (int k = 0; k < P && q < R; ++k) {
    acc += cost[k];
    const int left = P - (k + 1);
    if (acc >= tot * q / R || left == R - q) p.cut[q++] = k + 1;
  }
  const int S0 = f.R_off[P];
  // boundary separators (compact vector B) and internal separator ranges (T positions)
  p.B_off.assign(R, 0);
  p.B_pos.assign(std::max(R - 1, 0), 0);
  for (int b = 0; b + 1 < R; ++b) {
    const int j = p.cut[b + 1] - 1;
    p.B_pos[b] = f.S_off[j] - S0;
    p.B_off[b + 1] = p.B_off[b] + (f.S_off[j + 1] - f.S_off[j]);
  }
  p.nB = p.B_off[R - 1];
  p.I0.assign(R, 0); p.I1.assign(R, 0);
  for (int b = 0; b < R; ++b) {
    const int a = p.cut[b], e = p.cut[b + 1];
    // internal separators S_a .. S_{e-2}
    p.I0[b] = (e - a >= 2) ? f.S_off[a] - S0 : 0;
    p.I1[b] = (e - a >= 2) ? f.S_off[e - 1] - S0 : 0;
  }
  const int a = p.cut[r], e = p.cut[r + 1];
  p.stage_lo = a; p.stage_hi = e;
  p.leaf_lo = f.L_off[a]; p.leaf_hi = f.L_off[e];
  p.R_lo = f.R_off[a]; p.R_hi = f.R_off[e];
  // local separator rows: left boundary S_{a-1} .. right boundary S_{e-1} (internal index)
  p.sep_lo = (a > 0) ? f.S_off[a - 1] : f.S_off[a < P - 1 ? a : P - 1];
  p.sep_hi = (e < P) ? f.S_off[e] : f.S_off[P - 1];
  if (P == 1) p.sep_lo = p.sep_hi = S0;
  // owned rows: the right boundary is owned by the left rank (this one)
  p.own_sep_lo = (a > 0) ? f.S_off[a] : p.sep_lo;
  p.own_sep_hi = p.sep_hi;
  p.adj_lo = (r > 0) ? p.B_off[r - 1] : 0;
  p.adj_hi = (r < R - 1) ? p.B_off[r + 1] : p.nB;
  return STROM_OK;
}

// T = K'_SS - sum_k F_k^T F_k (lower and upper filled), from the host dense factors.
void host_schur_T(const Factor &f, Dense &T) {
  T = f.T0;
  for (int k = 0; k < f.P; ++k)
    if (!f.stage_cmap[k].empty() && f.R_off[k + 1] > f.R_off[k])
      dense_sub_AtA(T, f.F[f.stage_uid[k]], f.stage_cmap[k]);
}

namespace {
// rows of T's boundary b (T positions) -> compact offset
int bpos_to_T(const PartPlan &p, int c) {   // compact boundary index -> T position
  int b = 0;
  while (b + 1 < (int)p.B_pos.size() && p.B_off[b + 1] <= c) ++b;
  return p.B_pos[b] + (c - p.B_off[b]);
}
}  // namespace

strom_status host_factor_partition(const Factor &f, const PartPlan &p, PartFactor &pf) {
  Dense T;
  host_schur_T(f, T);
  const int R = p.R;
  pf.LIinv.assign(R, Dense());
  pf.W.assign(R, Dense());
  Dense Tt;                                   // T~ = T_BB - sum_q T_BI^q W^q
  Tt.rows = Tt.cols = p.nB;
  Tt.a.assign((size_t)p.nB * p.nB, 0.0);
  for (int c = 0; c < p.nB; ++c)
    for (int d = 0; d < p.nB; ++d) Tt.row(c)[d] = T.row(bpos_to_T(p, c))[bpos_to_T(p, d)];
  for (int q = 0; q < R; ++q) {
    const int i0 = p.I0[q], ni = p.I1[q] - p.I0[q];
    const int alo = (q > 0) ? p.B_off[q - 1] : 0, ahi = (q < R - 1) ? p.B_off[q + 1] : p.nB;
    const int wb = ahi - alo;
    if (ni == 0) continue;
    Dense L; L.rows = L.cols = ni; L.a.resize((size_t)ni * ni);
    for (int i = 0; i < ni; ++i)
      for (int j = 0; j < ni; ++j) L.row(i)[j] = T.row(i0 + i)[i0 + j];
    if (!dense_cholesky_lower(L)) {
      set_error("partition: non-positive pivot in an internal separator block");
      return STROM_EFACTOR;
    }
    dense_trinv_lower(L, pf.LIinv[q]);
    // W = L^{-T} L^{-1} T_IB
    Dense TIB; TIB.rows = ni; TIB.cols = wb; TIB.a.resize((size_t)ni * wb);
    for (int i = 0; i < ni; ++i)
      for (int c = 0; c < wb; ++c) TIB.row(i)[c] = T.row(i0 + i)[bpos_to_T(p, alo + c)];
    Dense Z;
    dense_gemm_lowertri(pf.LIinv[q], TIB, Z);          // L^{-1} T_IB
    Dense &W = pf.W[q];
    W.rows = ni; W.cols = wb; W.a.assign((size_t)ni * wb, 0.0);
    for (int i = 0; i < ni; ++i)                        // L^{-T} Z
      for (int k = i; k < ni; ++k) {
        const double l = pf.LIinv[q].row(k)[i];
        for (int c = 0; c < wb; ++c) W.row(i)[c] += l * Z.row(k)[c];
      }
    for (int c = 0; c < wb; ++c)
      for (int d = 0; d < wb; ++d) {
        double sdot = 0.0;
        for (int i = 0; i < ni; ++i) sdot += TIB.row(i)[c] * W.row(i)[d];
        Tt.row(alo + c)[alo + d] -= sdot;
      }
  }
  if (p.nB > 0) {
    if (!dense_cholesky_lower(Tt)) {
      set_error("partition: non-positive pivot in the reduced boundary system");
      return STROM_EFACTOR;
    }
    dense_trinv_lower(Tt, pf.LBinv);
  }
  return STROM_OK;
}

namespace {
// Phases P1-P3 of the solve restricted to rank p.r (host_solve's order): returns the
// rank's u (internal numbering; local rows only) and v.
void host_part_forward(const Factor &f, const PartPlan &p, const double *r_orig, std::vector<double> &rr,
                       std::vector<double> &u, std::vector<double> &v) {
  const int m = f.m, nL = f.nL, S0 = f.R_off[f.P];
  rr.assign(m, 0.0); u.assign(m, 0.0); v.assign(m, 0.0);
  // the rank's share of r: own leaf rows, own interior rows, own separators (the right
  // boundary belongs to the left rank)
  for (int i = p.leaf_lo; i < p.leaf_hi; ++i) rr[i] = r_orig[f.perm[i]];
  for (int i = p.R_lo; i < p.R_hi; ++i) rr[i] = r_orig[f.perm[i]];
  for (int i = p.own_sep_lo; i < p.own_sep_hi; ++i) rr[i] = r_orig[f.perm[i]];
  auto q_rows = [&](auto &&fn) {
    for (int i = p.R_lo; i < p.R_hi; ++i) fn(i);
    for (int i = p.sep_lo; i < p.sep_hi; ++i) fn(i);
  };
  q_rows([&](int q) {                                   // P1: u_Q = r_Q - G r_L
    double sum = rr[q];
    for (int64_t t = f.G_ptr[q - nL]; t < f.G_ptr[q - nL + 1]; ++t) sum -= f.G_val[t] * rr[f.G_col[t]];
    u[q] = sum;
  });
  for (int k = p.stage_lo; k < p.stage_hi; ++k) {      // P2: v_k = L_k^{-1} u_Rk
    const Dense &Li = f.Linv[f.stage_uid[k]];
    const int r0 = f.R_off[k];
    for (int i = 0; i < Li.rows; ++i) {
      double sum = 0.0;
      for (int j = 0; j <= i; ++j) sum += Li.row(i)[j] * u[r0 + j];
      v[r0 + i] = sum;
    }
  }
  for (int k = p.stage_lo; k < p.stage_hi; ++k) {      // P3: u_S -= F_k^T v_k (own stages)
    const Dense &F = f.F[f.stage_uid[k]];
    const int r0 = f.R_off[k], wl = f.stage_wl[k];
    for (int c = 0; c < F.cols; ++c) {
      const int si = (c < wl) ? f.S_off[k - 1] + c : f.S_off[k] + (c - wl);
      double sum = 0.0;
      for (int i = 0; i < F.rows; ++i) sum += F.row(i)[c] * v[r0 + i];
      u[si] -= sum;
    }
  }
  (void)S0;
}
}  // namespace

void host_part_begin(const Factor &f, const PartPlan &p, const PartFactor &pf, const double *r_orig,
                     double *send) {
  std::vector<double> rr, u, v;
  host_part_forward(f, p, r_orig, rr, u, v);
  const int S0 = f.R_off[f.P];
  for (int c = 0; c < p.nB; ++c) send[c] = 0.0;
  const int q = p.r, i0 = p.I0[q], ni = p.I1[q] - p.I0[q];
  for (int c = p.adj_lo; c < p.adj_hi; ++c) {
    double sum = u[S0 + bpos_to_T(p, c)];
    for (int i = 0; i < ni; ++i) sum -= pf.W[q].row(i)[c - p.adj_lo] * u[S0 + i0 + i];
    send[c] = sum;
  }
}

void host_part_end(const Factor &f, const PartPlan &p, const PartFactor &pf, const double *r_orig,
                   const double *recv, double *y_orig) {
  std::vector<double> rr, u, v;
  host_part_forward(f, p, r_orig, rr, u, v);
  const int m = f.m, nL = f.nL, S0 = f.R_off[f.P];
  std::vector<double> y(m, 0.0);
  // y_B = L~^{-T} L~^{-1} u~_B (replicated)
  const int nB = p.nB;
  std::vector<double> z(nB, 0.0), yB(nB, 0.0);
  for (int i = 0; i < nB; ++i) {
    double sum = 0.0;
    for (int j = 0; j <= i; ++j) sum += pf.LBinv.row(i)[j] * recv[j];
    z[i] = sum;
  }
  for (int i = 0; i < nB; ++i) {
    double sum = 0.0;
    for (int j = i; j < nB; ++j) sum += pf.LBinv.row(j)[i] * z[j];
    yB[i] = sum;
  }
  for (int c = 0; c < nB; ++c) y[S0 + bpos_to_T(p, c)] = yB[c];
  // y_I = T_II^{-1} u_I - W y_B,adj
  const int q = p.r, i0 = p.I0[q], ni = p.I1[q] - p.I0[q];
  if (ni > 0) {
    const Dense &Li = pf.LIinv[q];
    std::vector<double> t(ni), zi(ni);
    for (int i = 0; i < ni; ++i) {
      double sum = 0.0;
      for (int j = 0; j <= i; ++j) sum += Li.row(i)[j] * u[S0 + i0 + j];
      t[i] = sum;
    }
    for (int i = 0; i < ni; ++i) {
      double sum = 0.0;
      for (int j = i; j < ni; ++j) sum += Li.row(j)[i] * t[j];
      zi[i] = sum;
    }
    for (int i = 0; i < ni; ++i) {
      double sum = zi[i];
      for (int c = p.adj_lo; c < p.adj_hi; ++c) sum -= pf.W[q].row(i)[c - p.adj_lo] * yB[c];
      y[S0 + i0 + i] = sum;
    }
  }
  // P6: y_Rk = L_k^{-T} (v_k - F_k y_S,adj), own stages
  for (int k = p.stage_lo; k < p.stage_hi; ++k) {
    const Dense &Li = f.Linv[f.stage_uid[k]];
    const Dense &F = f.F[f.stage_uid[k]];
    const int r0 = f.R_off[k], nk = Li.rows, wl = f.stage_wl[k];
    std::vector<double> t(nk);
    for (int i = 0; i < nk; ++i) {
      double sum = v[r0 + i];
      for (int c = 0; c < F.cols; ++c) {
        const int si = (c < wl) ? f.S_off[k - 1] + c : f.S_off[k] + (c - wl);
        sum -= F.row(i)[c] * y[si];
      }
      t[i] = sum;
    }
    for (int i = 0; i < nk; ++i) {
      double sum = 0.0;
      for (int j = i; j < nk; ++j) sum += Li.row(j)[i] * t[j];
      y[r0 + i] = sum;
    }
  }
  // P7: y_L = K_LL^{-1} r_L - G^T y_Q, own leaves (groups never straddle stages)
  for (size_t g = 0; g + 1 < f.gptr.size(); ++g) {
    const int g0 = f.gptr[g], gs = f.gptr[g + 1] - g0;
    if (g0 < p.leaf_lo || g0 >= p.leaf_hi) continue;
    const double *Kinv = f.gKinv.data() + f.goff[g];
    for (int a = 0; a < gs; ++a) {
      double sum = 0.0;
      for (int c = 0; c < gs; ++c) sum += Kinv[a * gs + c] * rr[g0 + c];
      const int l = g0 + a;
      for (int64_t t = f.Gt_ptr[l]; t < f.Gt_ptr[l + 1]; ++t) sum -= f.Gt_val[t] * y[f.Gt_col[t]];
      y[l] = sum;
    }
  }
  (void)nL;
  // local rows only (others 0); boundary rows carry the replicated y_B
  for (int i = 0; i < m; ++i) y_orig[f.perm[i]] = 0.0;
  auto put = [&](int lo, int hi) { for (int i = lo; i < hi; ++i) y_orig[f.perm[i]] = y[i]; };
  put(p.leaf_lo, p.leaf_hi);
  put(p.R_lo, p.R_hi);
  put(p.sep_lo, p.sep_hi);
}

}  // namespace strom
