// Dense fp64 building blocks for the one-time factorisation of eps I + AA*
// (eq:strom:gpu:cholesky). Setup only, never on the hot path.
#include <cmath>

#include "host.h"

namespace strom {

// Left-looking Cholesky, row-major lower triangle, in place. Rows are
// contiguous so every inner product is a contiguous dot.
bool dense_cholesky_lower(Dense &A) {
  const int n = A.rows;
  bool ok = true;
  for (int j = 0; j < n && ok; ++j) {
    double *Lj = A.row(j);
    double d = Lj[j];
    for (int k = 0; k < j; ++k) d -= Lj[k] * Lj[k];
    if (!(d > 0.0) || !std::isfinite(d)) { ok = false; break; }
    const double ljj = std::sqrt(d);
    Lj[j] = ljj;
    const double inv = 1.0 / ljj;
#pragma omp parallel for schedule(static) if (n - j > 256)
    for (int i = j + 1; i < n; ++i) {
      double *Li = A.row(i);
      double s = Li[j];
      for (int k = 0; k < j; ++k) s -= Li[k] * Lj[k];
      Li[j] = s * inv;
    }
  }
  if (ok)
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) A.row(i)[j] = 0.0;
  return ok;
}

// X = L^{-1}, lower triangular, column by column (forward substitution on e_j).
void dense_trinv_lower(const Dense &L, Dense &X) {
  const int n = L.rows;
  X.rows = X.cols = n;
  X.a.assign((size_t)n * n, 0.0);
#pragma omp parallel
  {
    std::vector<double> x(n);
#pragma omp for schedule(dynamic, 8)
    for (int j = 0; j < n; ++j) {
      x[j] = 1.0 / L.row(j)[j];
      for (int i = j + 1; i < n; ++i) {
        const double *Li = L.row(i);
        double s = 0.0;
        for (int k = j; k < i; ++k) s += Li[k] * x[k];
        x[i] = -s / Li[i];
      }
      for (int i = j; i < n; ++i) X.row(i)[j] = x[i];
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
