"""ORACLE (test infrastructure only) -- sGS-ADMM, Algorithm 1 of PAPER.md:451-493.

Plain CPU fp64, step by step in the paper's order and notation:

  Step 1  r_s^{k+1/2} = b/sigma - A(X^k/sigma + S^k - C),  y^{k+1/2} = (eps I + AA*)^{-1} r_s
  Step 2  X_b = X^k + sigma (A* y^{k+1/2} - C),  S^{k+1} = (Pi_{Omega+}(X_b) - X_b)/sigma
  Step 3  r_s^{k+1} = b/sigma - A(X^k/sigma + S^{k+1} - C),  y^{k+1} = (eps I + AA*)^{-1} r_s
  Step 4  X^{k+1} = X^k + tau sigma (S^{k+1} + A* y^{k+1} - C)

Sub-steps with a plain definition use plain means:
  * A(X) and A*y: scipy CSR products with the matrix whose rows are svec(A_i)
    (PAPER.md:314, 439);
  * (eps I + AA*)^{-1} r: the eps-shifted normal matrix (eq:strom:gpu:cholesky,
    PAPER.md:587-591) factored once by SuperLU (a library sparse direct solve);
  * Pi_{Omega+}: per block, eigendecomposition X = Q W Q^T by LAPACK (numpy
    eigh), then Q max(0, W) Q^T (Higham 1988).
KKT residuals eta_p, eta_d, eta_g: eq:strom:sgsadmm:kkt-residual.

Readings: eps = eps_rel * max diag(AA*) (Q3), svec SDPT3
(Q4), cold start X = S = 0 (Q13), eta evaluated every iteration at
(X^{k+1}, y^{k+1}, S^{k+1}) (Q14), sigma policy (Q2) in `sigma_update`.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import sqrt
from typing import List, Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

_SQ2 = sqrt(2.0)


# ---------------------------------------------------------------------------
# svec <-> symmetric matrix (SDPT3: upper triangle column-wise, off-diag * sqrt2)
# ---------------------------------------------------------------------------
def _triu_colwise(n: int):
    r, c = [], []
    for j in range(n):
        for i in range(j + 1):
            r.append(i); c.append(j)
    return np.asarray(r), np.asarray(c)


_TRI_CACHE: dict = {}


def _tri(n: int):
    if n not in _TRI_CACHE:
        _TRI_CACHE[n] = _triu_colwise(n)
    return _TRI_CACHE[n]


def svec_to_mat(v: np.ndarray, n: int) -> np.ndarray:
    """smat: the symmetric matrix whose SDPT3 svec is v."""
    r, c = _tri(n)
    M = np.zeros(v.shape[:-1] + (n, n))
    w = np.where(r == c, v, v / _SQ2)
    M[..., r, c] = w
    M[..., c, r] = w
    return M


def mat_to_svec(M: np.ndarray) -> np.ndarray:
    n = M.shape[-1]
    r, c = _tri(n)
    v = M[..., r, c]
    return np.where(r == c, v, v * _SQ2)


def project_psd_block(M: np.ndarray) -> np.ndarray:
    """Pi_{S+}(X) = Q max(0, W) Q^T with X = Q W Q^T. Batched."""
    W, Q = np.linalg.eigh(M)
    return (Q * np.maximum(W, 0.0)[..., None, :]) @ np.swapaxes(Q, -1, -2)


# ---------------------------------------------------------------------------
@dataclass
class OracleConfig:
    sigma: float = 1.0            # sigma > 0; sigma_0 = 1 (Q2)
    tau: float = 1.618            # tau in (0, 2); reading Q1
    eps_rel: float = 1e-12        # eps = eps_rel * max diag(AA*) (Q3)
    eps: Optional[float] = None   # explicit eps overrides eps_rel
    sigma_period: int = 0         # 0 => fixed sigma (parity runs)
    sigma_ratio: float = 2.0
    sigma_factor: float = 1.2
    sigma_min: float = 1e-4
    sigma_max: float = 1e4


def sigma_update(sigma: float, it: int, eta_d: float, eta_x: float,
                 cfg: OracleConfig) -> float:
    """Residual-balancing sigma policy (reading Q2; PAPER.md:454 only says sigma > 0).

    sigma penalises the dual constraint A*y + S = C whose violation is eta_d; the
    matching ADMM dual residual is eta_x = ||X^{k+1} - Pi(X_b^{k+1})|| / (1 + ||X^{k+1}||),
    the distance of the multiplier X from the projected point (it scales with sigma).
    Every `sigma_period` completed iterations: eta_d > ratio * eta_x -> sigma *= factor;
    eta_x > ratio * eta_d -> sigma /= factor; clamped to [sigma_min, sigma_max].
    """
    if cfg.sigma_period <= 0 or it % cfg.sigma_period != 0:
        return sigma
    if eta_d > cfg.sigma_ratio * eta_x:
        sigma = min(sigma * cfg.sigma_factor, cfg.sigma_max)
    elif eta_x > cfg.sigma_ratio * eta_d:
        sigma = max(sigma / cfg.sigma_factor, cfg.sigma_min)
    return sigma


def kkt_residuals(AX: np.ndarray, b: np.ndarray, Aty: np.ndarray, S: np.ndarray,
                  C: np.ndarray, X: np.ndarray, y: np.ndarray):
    """(eta_p, eta_d, eta_g, <C,X>, <b,y>) per eq:strom:sgsadmm:kkt-residual."""
    eta_p = np.linalg.norm(AX - b) / (1.0 + np.linalg.norm(b))
    eta_d = np.linalg.norm(Aty + S - C) / (1.0 + np.linalg.norm(C))
    pobj = float(C @ X)
    dobj = float(b @ y)
    eta_g = abs(pobj - dobj) / (1.0 + abs(pobj) + abs(dobj))
    return float(eta_p), float(eta_d), float(eta_g), pobj, dobj


@dataclass
class Trace:
    iters: List[int] = field(default_factory=list)
    eta_p: List[float] = field(default_factory=list)
    eta_d: List[float] = field(default_factory=list)
    eta_g: List[float] = field(default_factory=list)
    pobj: List[float] = field(default_factory=list)
    dobj: List[float] = field(default_factory=list)
    sigma: List[float] = field(default_factory=list)
    eta_x: List[float] = field(default_factory=list)


class Oracle:
    """sGS-ADMM on one BlockSdp (duck-typed: block_n, block_offset, A_indptr,
    A_indices, A_data, b, C)."""

    def __init__(self, sdp, cfg: OracleConfig | None = None):
        self.cfg = cfg or OracleConfig()
        self.sdp = sdp
        m, n = int(sdp.b.shape[0]), int(sdp.block_offset[-1])
        self.m, self.n = m, n
        self.A = sp.csr_matrix((np.asarray(sdp.A_data, dtype=np.float64),
                                np.asarray(sdp.A_indices), np.asarray(sdp.A_indptr)),
                               shape=(m, n))
        self.At = self.A.T.tocsr()
        self.b = np.asarray(sdp.b, dtype=np.float64)
        self.C = np.asarray(sdp.C, dtype=np.float64)
        AAt = (self.A @ self.At).tocsc()
        self.eps = float(self.cfg.eps) if self.cfg.eps is not None else \
            float(self.cfg.eps_rel * AAt.diagonal().max())
        K = (AAt + self.eps * sp.identity(m, format="csc")).tocsc()
        self.K = K
        # eps I + AA* is SPD; SuperLU with symmetric-mode diagonal pivoting
        self._lu = spla.splu(K, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                             options=dict(SymmetricMode=True))
        # blocks grouped by order for batched projection
        bn = np.asarray(sdp.block_n)
        bo = np.asarray(sdp.block_offset)
        self.groups = {}
        for nb in sorted(set(bn.tolist())):
            idx = np.nonzero(bn == nb)[0]
            L = nb * (nb + 1) // 2
            cols = (bo[idx][:, None] + np.arange(L)[None, :]).astype(np.int64)
            self.groups[nb] = cols
        self.X = np.zeros(n); self.S = np.zeros(n); self.y = np.zeros(m)
        self.sigma = self.cfg.sigma
        self.it = 0
        self.trace = Trace()

    # --- the plain sub-steps --------------------------------------------
    def apply_A(self, X: np.ndarray) -> np.ndarray:
        """A(X) = (<A_i, X>)_i."""
        return self.A @ X

    def apply_At(self, y: np.ndarray) -> np.ndarray:
        """A*y = sum_l y_l A_l."""
        return self.At @ y

    def solve(self, r: np.ndarray) -> np.ndarray:
        """y = (eps I + AA*)^{-1} r."""
        return self._lu.solve(r)

    def project(self, X: np.ndarray) -> np.ndarray:
        """Pi_{Omega+}(X): per-block PSD projection."""
        out = np.empty_like(X)
        for nb, cols in self.groups.items():
            Mb = svec_to_mat(X[cols], nb)
            out[cols] = mat_to_svec(project_psd_block(Mb))
        return out

    # --- Algorithm 1 ------------------------------------------------------
    def set_start(self, X=None, y=None, S=None):
        self.X = np.zeros(self.n) if X is None else np.array(X, dtype=np.float64)
        self.S = np.zeros(self.n) if S is None else np.array(S, dtype=np.float64)
        self.y = np.zeros(self.m) if y is None else np.array(y, dtype=np.float64)
        self.it = 0
        self.trace = Trace()

    def iterate_once(self):
        """One pass of Steps 1-4. Returns a dict of the
        intermediates for parity tests."""
        A, b, C, sig, tau = self.A, self.b, self.C, self.sigma, self.cfg.tau
        X, S = self.X, self.S
        # Step 1 (eq:strom:sgsadmm:solve-y1)
        r1 = b / sig - self.apply_A(X / sig + S - C)
        y_half = self.solve(r1)
        # Step 2 (eq:strom:sgsadmm:solve-S)
        Xb = X + sig * (self.apply_At(y_half) - C)
        S_new = (self.project(Xb) - Xb) / sig
        # Step 3 (eq:strom:sgsadmm:solve-y2) -- note X^k, not X_b (Q27)
        r2 = b / sig - self.apply_A(X / sig + S_new - C)
        y_new = self.solve(r2)
        # Step 4 (eq:strom:sgsadmm:solve-X)
        Aty = self.apply_At(y_new)
        X_new = X + tau * sig * (S_new + Aty - C)
        self.X, self.S, self.y = X_new, S_new, y_new
        self.it += 1
        ep, ed, eg, po, do = kkt_residuals(self.apply_A(X_new), b, Aty, S_new, C, X_new, y_new)
        # diagnostic eta_x = ||X^{k+1} - Pi(X_b)|| / (1 + ||X^{k+1}||), Pi(X_b) = X_b + sigma S
        eta_x = float(np.linalg.norm(X_new - (Xb + sig * S_new)) / (1.0 + np.linalg.norm(X_new)))
        t = self.trace
        t.iters.append(self.it); t.eta_p.append(ep); t.eta_d.append(ed); t.eta_g.append(eg)
        t.pobj.append(po); t.dobj.append(do); t.sigma.append(sig)
        t.eta_x.append(eta_x)
        self.sigma = sigma_update(sig, self.it, ed, eta_x, self.cfg)
        return {"r1": r1, "y_half": y_half, "Xb": Xb, "S": S_new, "r2": r2, "y": y_new,
                "Aty": Aty, "X": X_new, "eta": (ep, ed, eg), "pobj": po, "dobj": do,
                "sigma_used": sig, "eta_x": eta_x}

    def iterate(self, iters: int):
        out = None
        for _ in range(iters):
            out = self.iterate_once()
        return out

    def solve_to_tol(self, tol: float, maxiter: int):
        """Iterate until eta = max(eta_p, eta_d, eta_g) <= tol or maxiter."""
        for _ in range(maxiter):
            out = self.iterate_once()
            if max(out["eta"]) <= tol:
                return self.it, True
        return self.it, False

    def residuals(self):
        Aty = self.apply_At(self.y)
        return kkt_residuals(self.apply_A(self.X), self.b, Aty, self.S, self.C, self.X, self.y)
