"""Certificate of suboptimality on top of the GPU solve (host post-processing).

Not on the sGS-ADMM hot path: this is the paper's layer L3,
run by the paper in Matlab with fmincon. The valid lower bound

    LB = <b,y> + sum_beta R_beta min(0, lambda_min((C - A*y)_beta))

is computed on the GPU by `strom_admm_lower_bound`. This module provides the upper
bound p_hat = <C, X(z_hat)> from the three-step extraction: top
eigenvector of each moment block M_k, normalised by its first entry, degree-one
entries -> z_bar, then a local solve of the POP from z_bar; and the refined gap

    xi = (p_hat - LB) / (1 + |p_hat| + |LB|)
"""
from __future__ import annotations

from math import sqrt

import numpy as np


def _block_matrix(svec: np.ndarray, n: int) -> np.ndarray:
    M = np.zeros((n, n))
    iu = np.triu_indices(n)
    # SDPT3 column-wise upper triangle: order (r, c) with c major
    order = np.lexsort((iu[0], iu[1]))
    r, c = iu[0][order], iu[1][order]
    w = np.where(r == c, svec, svec / sqrt(2.0))
    M[r, c] = w
    M[c, r] = w
    return M


def extract_zbar(sdp, X: np.ndarray, vtop=None) -> np.ndarray:
    """Steps one and two of the extraction heuristic. `vtop`: the top
    eigenvectors computed on the GPU (StromAdmm.extract(), strom_admm_extract); else
    LAPACK on the host."""
    pop = sdp.meta["pop"]
    bo = np.asarray(sdp.block_offset)
    acc = np.zeros(pop.d)
    cnt = np.zeros(pop.d)
    for k, I in enumerate(pop.cliques):
        beta = sdp.meta["mom_block"][k]
        nb = int(sdp.block_n[beta])
        if vtop is not None:
            q = np.asarray(vtop[beta])
        else:
            q = np.linalg.eigh(_block_matrix(X[bo[beta]:bo[beta + 1]], nb))[1][:, -1]
        v = q / q[0]
        for j, e in enumerate(sdp.meta["basis"][k]):
            if sum(e) == 1:
                var = int(np.argmax(e))
                acc[I[var]] += v[j]
                cnt[I[var]] += 1
    return acc / np.maximum(cnt, 1)


def pendulum_upper_bound(sdp, X: np.ndarray, maxiter: int = 200, u_start=None, vtop=None):
    """p_hat for the pendulum POP: controls of z_bar, then a local solve over the
    controls (rollouts satisfy x_0 = x_init, the dynamics and SO(2) exactly;
    |u| <= 1 and fc_k >= fc_min are the local solver's constraints)."""
    from scipy.optimize import minimize
    from strom_inputs.models import pendulum_rollout

    pop = sdp.meta["pop"]
    N = pop.N
    p = pop.meta["params"]
    th0, thd0 = pop.meta["theta0"], pop.meta["theta_dot0"]
    zbar = extract_zbar(sdp, X, vtop)
    u0 = np.clip(np.array([zbar[5 * k + 4] for k in range(N)]), -1.0, 1.0)
    if u_start is not None:   # keep the better of the extracted and the previous controls
        if pop.objective(pendulum_rollout(N, u_start, th0, thd0, p)) < pop.objective(pendulum_rollout(N, u0, th0, thd0, p)):
            u0 = np.asarray(u_start, dtype=np.float64)

    def rollout(u):
        return pendulum_rollout(N, u, th0, thd0, p)

    def margin(u):
        z = rollout(u)
        fs = z[[5 * k + 3 for k in range(1, N + 1)]]
        return 1.0 - fs ** 2 - p.fc_min ** 2

    res = minimize(lambda u: pop.objective(rollout(u)), u0, method="SLSQP",
                   bounds=[(-1.0, 1.0)] * N, constraints=[{"type": "ineq", "fun": margin}],
                   options={"maxiter": maxiter, "ftol": 1e-12})
    u = np.clip(res.x, -1.0, 1.0)
    if not np.all(margin(u) >= -1e-12):
        u = u0
    z_hat = rollout(u)
    feasible = bool(np.all(margin(u) >= -1e-9))
    return pop.objective(z_hat), z_hat, feasible


def pendulum_controls(z_hat: np.ndarray, N: int) -> np.ndarray:
    return np.array([z_hat[5 * k + 4] for k in range(N)])


def suboptimality_gap(p_hat: float, lb: float) -> float:
    return (p_hat - lb) / (1.0 + abs(p_hat) + abs(lb))
