/*
 * strom.h -- C-ABI of the B200-native sGS-ADMM hot path (libstrom.so).
 *
 * The library solves the standard multi-block SDP that STROM's sparse moment
 * relaxation produces (eq:strom:popsdp:standardsdp)
 *
 *     min <C, X>  s.t.  A(X) = b,  X = (X_1, ..., X_B) in Omega_+ = prod S^{n_beta}_+
 *
 * and its dual  max <b, y>  s.t.  A* y + S = C,  S in Omega_+  
 * with Algorithm 1 (sGS-ADMM):
 *
 *   Step 1  r = b/sigma - A(X/sigma + S - C),  y_half = (eps I + AA*)^{-1} r
 *   Step 2  X_b = X + sigma (A* y_half - C),   S = (Pi_{Omega+}(X_b) - X_b) / sigma
 *   Step 3  r = b/sigma - A(X/sigma + S - C),  y = (eps I + AA*)^{-1} r
 *   Step 4  X = X + tau sigma (S + A* y - C)
 *
 * terminating on eta = max(eta_p, eta_d, eta_g) <= tol (eq:strom:sgsadmm:kkt-residual,
 * PAPER.md:498-510). eps I + AA* is factored once at setup (eq:strom:gpu:cholesky,
 * PAPER.md:587-591); every per-iteration step runs in hand-written sm_100a
 * kernels on one device stream.
 *
 * Layout conventions
 *   svec   : SDPT3 symmetric vectorisation: upper triangle,
 *            column by column, off-diagonal entries multiplied by sqrt(2), so
 *            <A, B> = svec(A) . svec(B). Block beta occupies svec(n_beta) =
 *            n_beta (n_beta + 1) / 2 consecutive doubles; blocks are concatenated
 *            in the order given to strom_sdp_create ("sorted by clique",
 *            PAPER.md:570). n = sum_beta svec(n_beta).
 *   rows   : the m constraint rows keep the caller's numbering in every
 *            host-visible vector (b, y). Internally they are renumbered into
 *            factor order; that is invisible at this boundary.
 *   fp64   : all arithmetic and all buffers are IEEE double.
 *
 * Ownership: every input is copied at create/setup; the caller may free it on
 * return. Handles own all device memory. Output buffers are caller-allocated.
 * Threading: calls on one handle are not thread-safe; distinct handles are
 * independent. Errors: every call returns a strom_status; strom_last_error()
 * returns a thread-local message describing the last failure.
 */
#ifndef STROM_H
#define STROM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  STROM_OK = 0,
  STROM_MAXITER = 1,      /* status, not an error: maxiter reached before tol   */
  STROM_EINVAL = -1,      /* bad argument / shape / non-chain structure         */
  STROM_ENOMEM = -2,      /* host or device allocation failed                   */
  STROM_EFACTOR = -3,     /* non-positive pivot factoring eps I + AA*           */
  STROM_EEIG = -4,        /* Jacobi eigensolver did not converge                */
  STROM_EDIVERGED = -5,   /* NaN/Inf in the iterate                             */
  STROM_ECUDA = -6,       /* CUDA runtime error (message in strom_last_error)   */
  STROM_ENCCL = -7,       /* NCCL error                                         */
  STROM_ENOTIMPL = -8     /* feature not built in this version                  */
} strom_status;

typedef struct strom_sdp strom_sdp;    /* immutable problem data, host side      */
typedef struct strom_admm strom_admm;  /* solver state bound to device + stream  */

/* One PSD block X_beta of order n. `stage` is its clique
 * index k (0-based) in the chain (Definition 1); blocks must be
 * given in non-decreasing stage order and every constraint row may touch blocks
 * of at most two adjacent stages (the chain-like pattern of Fig. 1 / PAPER.md:415).
 * A_beta, the columns of A on this block, is CSR over the `nrows` rows that touch
 * the block: rows[nrows] strictly ascending global row ids in [0, m),
 * rowptr[nrows + 1] (rowptr[0] = 0), col[] svec index within the block in
 * [0, svec(n)), val[] the coefficient of svec(A_i). C_svec[svec(n)] is the dense
 * svec of the objective block C_beta. */
typedef struct {
  int32_t n;
  int32_t stage;
  int32_t nrows;
  const int32_t *rows;
  const int64_t *rowptr;
  const int32_t *col;
  const double *val;
  const double *C_svec;
} strom_block;

/* Copies and validates the SDP. b[m] is the right-hand side.
 * EINVAL on: nblocks <= 0, m <= 0, n_beta <= 0, rows not ascending / out of
 * range, col out of range, stages decreasing, a row touching non-adjacent stages. */
strom_status strom_sdp_create(strom_sdp **out, int32_t nblocks, const strom_block *blocks,
                              int32_t m, const double *b);
void strom_sdp_destroy(strom_sdp *sdp);
/* n (total svec length) and m of a created SDP. */
strom_status strom_sdp_dims(const strom_sdp *sdp, int64_t *n, int32_t *m, int32_t *nblocks);

/* Algorithm parameters and the sigma policy (reading Q2). */
typedef struct {
  double sigma;          /* sigma > 0 (initial value)                                 */
  double tau;            /* tau in (0, 2)                                             */
  double eps_rel;        /* eps = eps_rel * max_i (AA*)_ii when eps <= 0 (reading Q3) */
  double eps;            /* explicit eps > 0 overrides eps_rel                        */
  int32_t sigma_period;  /* 0 = fixed sigma; else rebalance every period iterations  */
  double sigma_ratio;    /* rebalance when eta_d / eta_x leaves [1/ratio, ratio]      */
  double sigma_factor;   /* multiplicative sigma step                                 */
  double sigma_min, sigma_max;
  int32_t check_every;   /* solve(): host polls the device status every K iterations  */
  int32_t eig_max_sweeps;/* Jacobi sweep cap (reading Q25)                            */
  double eig_tol;        /* Jacobi rotates a column pair while |cos| > max(eig_tol, 4nu) */
  int32_t eig_warm;      /* 1 = start Jacobi from the previous iteration's eigenbasis */
  int32_t eig_cold_every;/* > 0: cold Jacobi start every this many iterations        */
} strom_admm_config;

void strom_admm_default_config(strom_admm_config *cfg);

/* Builds eps I + AA*, orders rows (leaf pairs, stage interiors, separators),
 * factors once (eq:strom:gpu:cholesky; dense blocks on the device at setup) and uploads
 * everything to `device`. `cuda_stream` is a cudaStream_t (NULL = the handle creates its
 * own), e.g. a torch.cuda.Stream().cuda_stream.
 * Multi-GPU (nranks > 1, one process per GPU, every rank passes the same SDP and the same
 * 128-byte NCCL unique id from strom_nccl_get_unique_id on rank 0): horizon partition
 * (the paper distributes the moment blocks over GPUs).
 * Rank r owns the contiguous stage range [cut_r, cut_{r+1}) (balanced by sum n_beta^3):
 * its blocks (K-EIG, the X update), leaf and interior rows and the separators between its
 * stages. The separator S_j at a cut couples two ranks; each rank eliminates its own rows
 * down to these boundary separators, so a solve needs ONE sum over ranks (NCCL allreduce)
 * of the boundary right-hand side, after which every rank solves the small reduced
 * boundary system redundantly; a third allreduce per iteration carries the boundary rows'
 * A X partials and the six residual sums, so every rank takes the same eta / sigma /
 * termination decision. The three allreduces are captured in the iteration graph.
 * strom_admm_get / get_device / lower_bound / extract are collective on a partitioned
 * handle (every rank calls them; they gather the iterate and return it in full on every
 * rank). EINVAL if nranks > 1 without an id or nranks > number of stages; ENCCL on
 * communicator errors.
 * Starts cold: X = S = 0 (reading Q13). */
strom_status strom_admm_setup(strom_admm **out, const strom_sdp *sdp, const strom_admm_config *cfg,
                              int device, void *cuda_stream, const void *nccl_unique_id,
                              int rank, int nranks);
void strom_admm_destroy(strom_admm *h);

/* New sigma, tau, sigma policy and eigensolver settings for a set-up handle (eps and
 * check_every stay: the factor and the captured graphs depend on them). Takes effect at
 * the next strom_admm_set_start. EINVAL on an invalid sigma / tau. */
strom_status strom_admm_reconfigure(strom_admm *h, const strom_admm_config *cfg);

/* Warm start (Algorithm 1 input X^0, S^0). Host buffers of full
 * length (X_svec[n], y[m], S_svec[n]); NULL means zeros. Resets the iteration
 * counter and sigma to cfg.sigma. */
strom_status strom_admm_set_start(strom_admm *h, const double *X_svec, const double *y,
                                  const double *S_svec);
/* Same with device pointers on the handle's device (e.g. torch CUDA tensors). */
strom_status strom_admm_set_start_device(strom_admm *h, const double *dX, const double *dy,
                                         const double *dS);

/* Exactly `iters` iterations of Steps 1-4, no tolerance test (eta still
 * evaluated every iteration). Asynchronous on the handle's stream. */
strom_status strom_admm_iterate(strom_admm *h, int64_t iters);

/* Iterates until eta <= tol (checked every iteration on the device, polled by
 * the host every check_every iterations) or maxiter. Returns STROM_OK or
 * STROM_MAXITER; *iters_done = iterations performed by this call. */
strom_status strom_admm_solve(strom_admm *h, double tol, int64_t maxiter, int64_t *iters_done);

/* KKT residuals at the current iterate (X^k, y^k, S^k). */
typedef struct {
  int64_t iter;
  double eta_p, eta_d, eta_g;   /* eq:strom:sgsadmm:kkt-residual            */
  double pobj, dobj;            /* <C, X>, <b, y>                           */
  double sigma;                 /* sigma that produced this iterate         */
  double eta_x;                 /* ||X - Pi(X_b)|| / (1 + ||X||), diagnostic */
  int64_t eig_sweeps;           /* Jacobi sweeps summed over blocks since setup */
  int64_t iter_eta[3];          /* first iteration (since set_start) with eta <= 1e-4,
                                   1e-5, 1e-6, tracked on the device; 0 = not reached */
} strom_residuals;

/* Copies the iterate to host buffers (NULL = skip). Synchronises the stream. */
strom_status strom_admm_get(strom_admm *h, double *X_svec, double *y, double *S_svec,
                            strom_residuals *res);
/* Device-to-device copy into caller device buffers (NULL = skip). Asynchronous. */
strom_status strom_admm_get_device(strom_admm *h, double *dX, double *dy, double *dS);

/* Valid lower bound LB = <b,y> + sum_beta R_beta min(0, lambda_min((C - A*y)_beta))
 * (eq:strom:sgsadmm:valid-lowerbound) at the current y, computed
 * on the device (A*y and an eigenvalues-only Jacobi). R_beta[nblocks] host array
 * (Theorem 2). lambda_min[nblocks] optional output: the computed
 * smallest eigenvalue of each block lowered by its error margin 3 n_beta u ||Z_beta||_F
 * (Z = C - A*y, u = 2^-53), so the bound is never overstated by rounding. EEIG when a
 * block hit the Jacobi sweep cap (a capped run overestimates lambda_min; no bound is
 * returned). The iterate and the solver state (done flag, residuals) are unchanged. */
strom_status strom_admm_lower_bound(strom_admm *h, const double *R_beta, double *lb,
                                    double *lambda_min);

/* Extraction data for the certificate ("extract a feasible solution
 * from the eigenvectors of the moment matrices"), computed on the device at the current
 * X by the K-EIG kernels in a cold eigendecomposition mode: for every block beta,
 * lam12[2 beta] >= lam12[2 beta + 1] are the two largest eigenvalues of X_beta (their
 * ratio is the tightness test: a rank-one moment matrix has lambda_2 = 0), and, when vtop
 * is non-NULL, vtop[off_beta .. off_beta + n_beta) the unit eigenvector of the largest,
 * sign fixed so that its first entry is >= 0 (off_beta = sum of n over earlier blocks;
 * vtop holds sum_beta n_beta doubles). Host buffers owned by the caller; the iterate and
 * the solver state are unchanged. EINVAL on NULL handle/lam12. */
strom_status strom_admm_extract(strom_admm *h, double *lam12, double *vtop);

/* ---- batched instances (NEXT-2: the paper's grid of initial states) ----
 * `count` single-GPU handles on one device, each with its own stream, iterated by ONE CUDA
 * graph in which every handle's `iters_per_launch` iterations form an independent branch
 * (a fork on `cuda_stream`, NULL = own stream, and a join), so the instances run
 * concurrently and fill the SMs one instance leaves idle. Every handle keeps its own
 * iterate, residuals, sigma and termination; results equal separate runs bitwise. The
 * handles stay owned by the caller and must outlive the batch; strom_admm_get etc. on a
 * handle are ordered after the batch's work. EINVAL on mixed devices, shared streams or
 * partitioned (multi-GPU) handles. */
typedef struct strom_batch strom_batch;
strom_status strom_batch_create(strom_batch **out, strom_admm *const *handles, int32_t count,
                                int32_t iters_per_launch, void *cuda_stream);
void strom_batch_destroy(strom_batch *b);
/* Exactly `iters` iterations of every instance (a multiple of iters_per_launch). Async. */
strom_status strom_batch_iterate(strom_batch *b, int64_t iters);
/* Iterates until every instance has eta <= tol (each stops at its own first such
 * iteration) or maxiter; iters_done[count] (nullable) = iterations each instance performed,
 * converged[count] (nullable) = 1 where eta <= tol was reached. OK when all converged,
 * MAXITER otherwise, EDIVERGED on NaN/Inf in any instance. */
strom_status strom_batch_solve(strom_batch *b, double tol, int64_t maxiter, int64_t *iters_done,
                               int32_t *converged);

/* Wall-clock milliseconds of the setup phases of a handle: ms[0] host factorisation
 * (build_factor: AA*, leaf groups, K'), ms[1] uploads, ms[2] device dense factors
 * (cuSOLVER/cuBLAS), ms[3] eigensolver classes and state, ms[4] graph capture. */
strom_status strom_admm_setup_times(const strom_admm *h, double *ms);

/* Number of kernel launches one iteration issues (for launch accounting). */
int32_t strom_admm_launches_per_iter(const strom_admm *h);
/* Size of the factor data on the device in bytes, and unique dense factors. */
strom_status strom_admm_factor_info(const strom_admm *h, int64_t *device_bytes,
                                    int32_t *n_leaf_rows, int32_t *n_sep_rows,
                                    int32_t *n_unique_dense);

/* Per-kernel device times (ms) of the instrumented iteration: the last iteration
 * of the most recent check_every-iteration graph launch carries CUDA event
 * record nodes around each of its kernel launches (on the handle's stream).
 * Fills ms[i] and names[i] (static strings) for i < min(count, cap); returns the
 * number of launches per iteration, or a negative strom_status. */
int32_t strom_admm_kernel_times(strom_admm *h, double *ms, const char **names, int32_t cap);

/* Algorithmic work of one launch of the kernel marked `name` (a name returned by
 * strom_admm_kernel_times, e.g. "trsv_p2_stage_Linv", "update_X"): *bytes = the factor
 * entries it must read once (unique stage factors counted once) plus its input and output
 * vectors, *flops = its fp64 flops. The K-EIG classes ("eig_classN") are
 * not listed (their work is sum 10 n^3 over the class's blocks, computed by the caller).
 * STROM_EINVAL for a NULL argument or an unknown name. Reading only; no device work. */
strom_status strom_admm_kernel_work(strom_admm *h, const char *name, double *bytes, double *flops);

/* rank 0: fills the 128-byte NCCL unique id to broadcast (e.g. via torch.distributed). */
strom_status strom_nccl_get_unique_id(void *id128);
const char *strom_last_error(void);
const char *strom_version(void);

/* ---- test hooks (not part of the user contract) -----------------------------
 * Each runs one kernel family on the handle's device on host buffers. */
/* S_out = (Pi(X_b) - X_b) / sigma per block; also returns Pi(X_b) when non-NULL. */
strom_status strom_debug_project_psd(strom_admm *h, const double *Xb, double sigma,
                                     double *S_out, double *Pi_out);
/* Ax[m] = A(X), Aty[n] = A* y (either may be NULL). */
strom_status strom_debug_spmv(strom_admm *h, const double *X, double *AX,
                              const double *y, double *Aty);
/* y = (eps I + AA*)^{-1} r on the device (rows in caller numbering). */
strom_status strom_debug_solve(strom_admm *h, const double *r, double *y);
/* Same solve executed by the HOST from the setup factor (checks the setup
 * factorisation without a GPU; never used by the iteration). */
strom_status strom_debug_host_solve(const strom_sdp *sdp, const strom_admm_config *cfg,
                                    const double *r, double *y);
/* Host execution of the horizon-partitioned solve for rank `rank` of
 * `nranks` (CPU test of the partition logic, e.g. under a gloo process group). nB (out,
 * nullable) = number of boundary separator rows. send != NULL: the rank's partial boundary
 * right-hand side u~_B^r (nB doubles) for y = (eps I + AA*)^{-1} r; recv && y: from the
 * summed u~_B (recv, nB) the rank's rows of y (caller numbering; rows the rank does not
 * hold are 0, boundary rows carry the replicated y_B). r is the full right-hand side. */
strom_status strom_debug_host_part(const strom_sdp *sdp, const strom_admm_config *cfg, int32_t nranks,
                                   int32_t rank, const double *r, double *send, const double *recv,
                                   double *y, int32_t *nB);
/* eps actually used by a handle. */
double strom_debug_eps(const strom_admm *h);
/* In-process "virtual ranks": nranks handles of the same SDP on one device, made by
 * strom_debug_setup_virtual (rank r of nranks), play the ranks of the multi-GPU mode with
 * the same kernels; each sum over ranks is a device kernel instead of an NCCL allreduce.
 * link: register the peers; iterate: `iters` lock-step iterations of all handles. */
strom_status strom_debug_setup_virtual(strom_admm **out, const strom_sdp *sdp, const strom_admm_config *cfg,
                                       int device, void *cuda_stream, int rank, int nranks);
strom_status strom_debug_link_virtual(strom_admm **handles, int32_t nranks, const strom_sdp *sdp);
strom_status strom_debug_iterate_virtual(strom_admm **handles, int32_t nranks, int64_t iters);

#ifdef __cplusplus
}
#endif
#endif /* STROM_H */
