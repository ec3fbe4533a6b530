// Dense fp64 building blocks for the one-time factorisation of eps I + AA*
// (eq:strom:gpu:cholesky). Setup only, never on the hot path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "host.h"

namespace strom {

// Blocked left-looking Cholesky, row-major lower triangle, in place: for each block of
// kB columns, (1) the rows at and below it subtract the contributions of all earlier
// columns (one pass over each row's left part per block, contiguous dots), (2) the
// diagonal block is factored, (3) the rows below solve against it. Reads every row's left
// part n/kB times instead of n times.
bool dense_cholesky_lower(Dense &A) {
  const int n = A.rows;
  constexpr int kB = 64;
  for (int J0 = 0; J0 < n; J0 += kB) {
    const int J1 = std::min(n, J0 + kB), jb = J1 - J0;
    // (1) A[i][J0:J1] -= L[i][0:J0] . L[j][0:J0] for j in the block, i >= J0
#pragma omp parallel for schedule(dynamic, 16) if (n - J0 > 128)
    for (int i = J0; i < n; ++i) {
      double *Li = A.row(i);
      const int jmax = std::min(J1, i + 1);
      for (int j = J0; j < jmax; ++j) {
        const double *Lj = A.row(j);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int k = 0;
        for (; k + 3 < J0; k += 4) {
          s0 += Li[k] * Lj[k]; s1 += Li[k + 1] * Lj[k + 1]; s2 += Li[k + 2] * Lj[k + 2]; s3 += Li[k + 3] * Lj[k + 3];
        }
        for (; k < J0; ++k) s0 += Li[k] * Lj[k];
        Li[j] -= (s0 + s1) + (s2 + s3);
      }
    }
    // (2) factor the diagonal block (left-looking inside the block)
    for (int j = J0; j < J1; ++j) {
      double *Lj = A.row(j);
      double d = Lj[j];
      for (int k = J0; k < j; ++k) d -= Lj[k] * Lj[k];
      if (!(d > 0.0) || !std::isfinite(d)) return false;
      const double ljj = std::sqrt(d);
      Lj[j] = ljj;
      const double inv = 1.0 / ljj;
      for (int i = j + 1; i < J1; ++i) {
        double *Li = A.row(i);
        double s = Li[j];
        for (int k = J0; k < j; ++k) s -= Li[k] * Lj[k];
        Li[j] = s * inv;
      }
    }
    // (3) rows below: L[i][J0:J1] = A[i][J0:J1] L_JJ^{-T} (forward substitution per row)
#pragma omp parallel for schedule(static) if (n - J1 > 128)
    for (int i = J1; i < n; ++i) {
      double *Li = A.row(i);
      for (int j = J0; j < J1; ++j) {
        const double *Lj = A.row(j);
        double s = Li[j];
        for (int k = J0; k < j; ++k) s -= Li[k] * Lj[k];
        Li[j] = s / Lj[j];
      }
    }
    (void)jb;
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A.row(i)[j] = 0.0;
  return true;
}

// X = L^{-1}, lower triangular: forward substitution on e_j, eight columns per pass so that
// each row of L is read once per eight columns.
void dense_trinv_lower(const Dense &L, Dense &X) {
  const int n = L.rows;
  X.rows = X.cols = n;
  X.a.assign((size_t)n * n, 0.0);
  constexpr int kC = 8;
#pragma omp parallel
  {
    std::vector<double> x((size_t)n * kC);
#pragma omp for schedule(dynamic, 1)
    for (int j0 = 0; j0 < n; j0 += kC) {
      const int nc = std::min(kC, n - j0);
      // x[i * kC + c]: component i of column j0 + c (zero above the diagonal)
      std::fill(x.begin(), x.end(), 0.0);
      for (int i = j0; i < n; ++i) {
        const double *Li = L.row(i);
        double s[kC] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = j0; k < i; ++k) {
          const double l = Li[k];
          const double *xk = &x[(size_t)k * kC];
          for (int c = 0; c < kC; ++c) s[c] += l * xk[c];
        }
        for (int c = 0; c < nc; ++c) {
          const int j = j0 + c;
          x[(size_t)i * kC + c] = i < j ? 0.0 : (i == j ? 1.0 / Li[i] : -s[c] / Li[i]);
        }
      }
      for (int i = j0; i < n; ++i)
        for (int c = 0; c < nc; ++c)
          if (i >= j0 + c) X.row(i)[j0 + c] = x[(size_t)i * kC + c];
    }
  }
}

// F = Linv * B with Linv lower triangular (n x n), B (n x w).
void dense_gemm_lowertri(const Dense &Linv, const Dense &B, Dense &F) {
  const int n = Linv.rows, w = B.cols;
  F.rows = n; F.cols = w;
  F.a.assign((size_t)n * w, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
  for (int i = 0; i < n; ++i) {
    double *Fi = F.row(i);
    const double *Li = Linv.row(i);
    for (int k = 0; k <= i; ++k) {
      const double l = Li[k];
      if (l == 0.0) continue;
      const double *Bk = B.row(k);
      for (int c = 0; c < w; ++c) Fi[c] += l * Bk[c];
    }
  }
}

// T[cmap[a], cmap[b]] -= sum_i F[i][a] F[i][b]
void dense_sub_AtA(Dense &T, const Dense &F, const std::vector<int32_t> &cmap) {
  const int n = F.rows, w = F.cols;
  Dense Ft; Ft.rows = w; Ft.cols = n; Ft.a.resize((size_t)w * n);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < w; ++c) Ft.row(c)[i] = F.row(i)[c];
#pragma omp parallel for schedule(dynamic, 4)
  for (int a = 0; a < w; ++a) {
    const double *fa = Ft.row(a);
    for (int b2 = 0; b2 < w; ++b2) {
      const double *fb = Ft.row(b2);
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += fa[i] * fb[i];
      T.row(cmap[a])[cmap[b2]] -= s;
    }
  }
}

}  // namespace strom
