// Host-side data structures of libstrom (internal; not part of the C-ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/strom.h"

namespace strom {

void set_error(const std::string &msg);

// Immutable problem data (strom_sdp), assembled into a global row CSR.
struct Sdp {
  int32_t nblocks = 0, m = 0, nstages = 0;
  int64_t n = 0;
  std::vector<int32_t> bn, bstage;
  std::vector<int64_t> boff;            // svec offset per block, nblocks + 1
  std::vector<int64_t> rowptr;          // m + 1
  std::vector<int32_t> col;             // global svec column
  std::vector<double> val;
  std::vector<double> b, C;
};

// Row-major dense matrix.
struct Dense {
  int32_t rows = 0, cols = 0;
  std::vector<double> a;
  double *row(int i) { return a.data() + (int64_t)i * cols; }
  const double *row(int i) const { return a.data() + (int64_t)i * cols; }
};

// The factorisation of eps I + AA* in "leaf / stage-interior / separator" form
// (DESIGN.md §K-TRSV). Internal row order: [leaf rows grouped][R_0]...[R_{P-1}][S_0]...[S_{P-2}].
struct Factor {
  double eps = 0.0;
  int32_t m = 0, P = 0;
  std::vector<int32_t> perm;   // internal -> original row
  std::vector<int32_t> iperm;  // original -> internal
  // leaf groups (rows [0, nL))
  int32_t nL = 0;
  std::vector<int32_t> gptr;   // ngroups + 1, internal row offsets
  std::vector<int64_t> goff;   // offsets into gKinv (g*g each)
  std::vector<double> gKinv;   // K_g^{-1}, row-major g x g
  std::vector<int32_t> L_off;  // P + 1: leaf rows of stage k are [L_off[k], L_off[k+1])
  // G = K_QL K_LL^{-1}: CSR over Q rows (q - nL), columns = leaf internal index
  std::vector<int64_t> G_ptr;
  std::vector<int32_t> G_col;
  std::vector<double> G_val;
  // G^T: CSR over leaf rows, columns = absolute internal index of Q rows
  std::vector<int64_t> Gt_ptr;
  std::vector<int32_t> Gt_col;
  std::vector<double> Gt_val;
  // stage interiors R_k = [R_off[k], R_off[k+1]) ; separators S_j = [S_off[j], S_off[j+1])
  std::vector<int32_t> R_off;  // P + 1
  std::vector<int32_t> S_off;  // P (S_0 .. S_{P-2}); S_off[0] = R_off[P]
  // unique dense stage blocks (inputs of the dense backend)
  std::vector<Dense> uK;       // K'_{R_k R_k}
  std::vector<Dense> uB;       // K'_{R_k, [S_{k-1} S_k]}
  Dense T0;                    // K'_SS
  std::vector<std::vector<int32_t>> stage_cmap;
  // unique dense stage factors (host backend output)
  std::vector<Dense> Linv;     // lower-triangular L_k^{-1} (n_k x n_k)
  std::vector<Dense> F;        // L_k^{-1} K'_{R_k, [S_{k-1} S_k]}  (n_k x (wl + wr))
  std::vector<int32_t> stage_uid;       // stage -> unique factor id
  std::vector<int32_t> stage_wl, stage_wr;
  Dense LTinv;                 // lower-triangular L_T^{-1} (|S| x |S|)
  int32_t nS() const { return m - (R_off.empty() ? 0 : R_off.back()); }
};

// Horizon partition (partition.cpp): rank r of R owns stages
// [cut[r], cut[r+1]). Separator positions are 0-based in T (= internal index - S0).
struct PartPlan {
  int32_t R = 1, r = 0;
  std::vector<int32_t> cut;            // R + 1 stage cuts
  std::vector<int32_t> B_off;          // R: compact offset of boundary b (b < R-1); B_off[R-1] = nB
  std::vector<int32_t> B_pos;          // R - 1: T position of boundary b (separator cut[b+1]-1)
  int32_t nB = 0;
  std::vector<int32_t> I0, I1;         // per rank: internal separators, T positions [I0, I1)
  // this rank (internal row indices)
  int32_t stage_lo = 0, stage_hi = 0, leaf_lo = 0, leaf_hi = 0, R_lo = 0, R_hi = 0;
  int32_t sep_lo = 0, sep_hi = 0;      // local separator rows incl. both boundaries
  int32_t own_sep_lo = 0, own_sep_hi = 0;   // owned separator rows (right boundary owned)
  int32_t adj_lo = 0, adj_hi = 0;      // compact range of the adjacent boundaries
};
struct PartFactor {                    // host dense partition factors (tests)
  std::vector<Dense> LIinv;            // per rank: (T_II^q)^{-1} Cholesky factor inverse
  std::vector<Dense> W;                // per rank: (T_II^q)^{-1} T_IB^q, |I_q| x |adjacent B|
  Dense LBinv;                         // reduced boundary system L~^{-1}
};

strom_status build_sdp(Sdp &s, int32_t nblocks, const strom_block *blocks, int32_t m,
                       const double *b);
strom_status build_factor(const Sdp &s, double eps_rel, double eps_abs, Factor &f);
strom_status host_factor_dense(Factor &f);
// Host execution of the factored solve (test hook / reference for the device phases).
void host_solve(const Factor &f, const double *r_orig, double *y_orig);

strom_status make_plan(const Sdp &s, const Factor &f, int R, int r, PartPlan &p);
void host_schur_T(const Factor &f, Dense &T);
strom_status host_factor_partition(const Factor &f, const PartPlan &p, PartFactor &pf);
void host_part_begin(const Factor &f, const PartPlan &p, const PartFactor &pf, const double *r_orig,
                     double *send);
void host_part_end(const Factor &f, const PartPlan &p, const PartFactor &pf, const double *r_orig,
                   const double *recv, double *y_orig);

// dense kernels (dense.cpp)
bool dense_cholesky_lower(Dense &A);           // in place, lower triangle; false on pivot <= 0
void dense_trinv_lower(const Dense &L, Dense &X);
void dense_gemm_lowertri(const Dense &Linv, const Dense &B, Dense &F);  // F = Linv * B
void dense_sub_AtA(Dense &T, const Dense &F, const std::vector<int32_t> &cmap);  // T[cmap,cmap] -= F^T F

}  // namespace strom
