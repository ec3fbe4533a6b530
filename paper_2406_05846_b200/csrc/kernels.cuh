// sm_100a kernels of the sGS-ADMM hot path (Algorithm 1).
// All arithmetic fp64. Every kernel reads sigma/tau from device memory so a
// captured CUDA graph stays valid when the sigma policy changes sigma, and
// returns immediately when the device `done` flag is set (solve-to-tol).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace strom {

struct DevState {          // scalars living on the device
  double sigma, tau, eps;
  double tol;              // < 0 => never stop (iterate())
  double normb, normC;
  int64_t iter;            // completed iterations of this run
  int32_t done;            // 1 => converged; kernels become no-ops
  int32_t eig_fail;        // Jacobi exceeded its sweep cap (block id + 1)
  int32_t nan_flag;
  int32_t sigma_period;
  int32_t eig_warm_valid;  // 1 once every block has a stored eigenbasis
  int32_t w_valid;         // 1 when RhsArgs::w holds AC - A S for the current S
  unsigned long long eig_sweeps;   // diagnostic: Jacobi sweeps summed over blocks
  uint32_t ticket;         // CTA arrival counter of the fused residual reduction
  double sigma_ratio, sigma_factor, sigma_min, sigma_max;
  // residuals of the latest completed iterate
  double eta_p, eta_d, eta_g, pobj, dobj, eta_x, sigma_used;
  int64_t iter_eta[3];     // first iteration with eta <= 1e-4, 1e-5, 1e-6 (0 = not yet)
};

// r_i = (b_i - AX_i) / sigma + (AC_i - (A S)_i) : Step 1/3 right-hand side
// (eq:strom:sgsadmm:solve-y1/-y2), formed on the fly by the solve phases; (A S)_i is a
// sparse row dot with the current S (no separate A S pass), skipped when S is null.
// Step 3 stores w_i = AC_i - (A S^{k+1})_i for every row it forms (wout); Step 1 of the
// next iteration has the same S and reads w instead of re-forming the dots (w, when
// DevState::w_valid).
struct RhsArgs {
  const double *b, *ax, *ac;
  const int64_t *Arp; const int32_t *Aci; const double *Av;
  const double *S;
  const double *w; double *wout;
};

// Per-row addressing of the solve phases, precomputed at setup so that no kernel walks a
// chain of dependent metadata loads (stage of a row -> factor id -> factor pointer ...)
// before its first data load. P3: separator row s -> the H^T rows of its two stages (null
// where the stage is another rank's) and their stage vector bases.
struct SepRowInfo { const double *h0, *h1; int32_t base0, base1, n0, n1; };
// P6'': interior row -> its H row, width and the two adjacent separator starts
struct IntRowInfo { const double *hrow; int32_t wk, wl, sl0, sr0; };
// P7: leaf row -> its group's first row, size and K_g^{-1} row offset
struct LeafRowInfo { int32_t g0, gs; int64_t kinv; };

struct SolveDev {
  int32_t m, nL, nQ, P, S0, nS;
  // leaf
  const int32_t *gptr; int32_t ngroups;
  const int64_t *goff; const double *gKinv;
  const int32_t *leaf_group;
  const int64_t *G_ptr; const int32_t *G_col; const double *G_val;
  const int64_t *Gt_ptr; const int32_t *Gt_col; const double *Gt_val;
  // stages
  const int32_t *R_off, *S_off, *stage_uid, *stage_wl, *stage_wr;
  // unique dense: Linv (lower, row-major), LinvT (= L^{-T}, row-major upper),
  // F (n_k x w), Ft (w x n_k)
  const double *const *Linv; const double *const *LinvT;
  const double *const *F; const double *const *Ft;
  const double *const *H; const double *const *Ht;   // H_k = L_k^{-T} F_k (n_k x w), H^T
  const int32_t *uid_n, *uid_w;
  // work vectors (internal order, length m)
  double *u, *v, *t, *z;
  // rows this handle works on (internal order). One GPU: everything. Horizon partition
  // (SURVEY.md §8(e)): the rank's leaves [L_lo, L_hi), interiors [R_lo, R_hi), separators
  // [Sl_lo, Sl_hi) incl. both boundaries, and its stages [stage_lo, stage_hi).
  int32_t L_lo, L_hi, R_lo, R_hi, Sl_lo, Sl_hi, stage_lo, stage_hi;
  const SepRowInfo *sep_info;      // [Sl_hi - Sl_lo]
  const IntRowInfo *int_info;      // [R_hi - R_lo]
  const LeafRowInfo *leaf_info;    // [L_hi - L_lo]
};

// Lower-triangular inverse (e.g. the separator L_T^{-1}, n x n) stored as its lower 64x64
// tiles (I >= J, tile-row-major order, each tile row-major, zero padded) for k_sep_tri, with
// the per-call partial products part[X][Y][64] and per-block arrival counters cnt[nT].
struct TriTiles {
  const double *tile; int32_t nT, n; double *part; unsigned *cnt;
  int32_t stream;               // tiles > 256 MB (HBM-streamed): evict-first loads
  int32_t yc;                   // input blocks (tiles) per CTA
  const int2 *work[2];          // yc > 1: per CTA of a pass (mode 0: L^{-1}, 1: L^{-T}): (X, first Y)
  int32_t nwork[2];             // CTAs of a pass
};

// Horizon-partitioned separator solve (partition.cpp) on the device, this rank's pieces.
struct PartDev {
  int32_t nB, adj_lo, adj_hi;          // boundary rows (compact), adjacent range
  int32_t I0, nI;                      // internal separators (T positions), count
  const int32_t *Bmap;                 // compact boundary index -> T position (nB)
  const double *W;                     // nI x wb row-major, W = T_II^{-1} T_IB
  const double *Wt;                    // wb x nI row-major
  TriTiles LI, LB;                     // (T_II)^{-1} factor tiles, reduced L~^{-1} tiles
  double *send, *recv, *tB, *yB, *zI, *zI2;   // nB, nB, nB, nB, nI, nI
};

}  // namespace strom
