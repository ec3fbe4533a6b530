"""ORACLE (test infrastructure only) -- the refined certificate of suboptimality.

  LB = <b,y> + sum_beta R_beta min{0, lambda_min((C - A*y)_beta)}
       (eq:inexact-lower-bound / eq:strom:sgsadmm:valid-lowerbound)
  xi = (<C, X(z_hat)> - LB) / (1 + |<C, X(z_hat)>| + |LB|)
       (eq:strom:sgsadmm:suboptimality-gap)
  z_hat: three-step extraction: top eigenvector v_k of M_k,
  v_k / v_k(1), degree-one entries -> z_bar, then a local solve of the POP from
  z_bar (the paper uses fmincon; here a control-parameterised SLSQP for the
  pendulum, whose rollouts satisfy every equality by construction).
R_beta: Theorem 2, read as in Q17 (provided by the input
generator as sdp.R_beta).
"""
from __future__ import annotations

import numpy as np

from .admm import svec_to_mat


def lower_bound(sdp, y: np.ndarray, Aty: np.ndarray, safety: bool = True):
    """Valid lower bound on p* from any y.

    lambda_min by LAPACK eigvalsh, minus a backward-error floor n*u*||Z||_F when
    `safety` (an eigenvalue computed by a backward-stable method is exact for a
    matrix within that distance, so the bound stays valid)."""
    Z = np.asarray(sdp.C) - Aty
    bo = np.asarray(sdp.block_offset)
    lam = np.empty(len(sdp.block_n))
    for beta, nb in enumerate(np.asarray(sdp.block_n)):
        Zb = svec_to_mat(Z[bo[beta]:bo[beta + 1]], int(nb))
        l0 = np.linalg.eigvalsh(Zb)[0]
        if safety:
            l0 -= nb * np.finfo(np.float64).eps * np.linalg.norm(Zb)
        lam[beta] = l0
    LB = float(np.asarray(sdp.b) @ y) + float(np.sum(np.asarray(sdp.R_beta) * np.minimum(0.0, lam)))
    return LB, lam


def suboptimality_gap(p_hat: float, LB: float) -> float:
    """xi of eq:strom:sgsadmm:suboptimality-gap."""
    return (p_hat - LB) / (1.0 + abs(p_hat) + abs(LB))


def extract_raw(sdp, X: np.ndarray) -> np.ndarray:
    """Steps one and two of the extraction heuristic: z_bar from
    the top eigenvectors of the moment blocks; shared variables averaged."""
    pop = sdp.meta["pop"]
    bo = np.asarray(sdp.block_offset)
    acc = np.zeros(pop.d); cnt = np.zeros(pop.d)
    for k, I in enumerate(pop.cliques):
        beta = sdp.meta["mom_block"][k]
        nb = int(sdp.block_n[beta])
        W, Q = np.linalg.eigh(svec_to_mat(X[bo[beta]:bo[beta + 1]], nb))
        v = Q[:, -1]
        v = v / v[0]
        basis = sdp.meta["basis"][k]
        for j, e in enumerate(basis):
            if sum(e) == 1:
                var = int(np.argmax(e))
                acc[I[var]] += v[j]; cnt[I[var]] += 1
    return acc / np.maximum(cnt, 1)


def extract_pendulum(sdp, X: np.ndarray, refine: bool = True):
    """z_hat and p_hat for the pendulum POP: extraction then a local solve over
    the controls (rollouts satisfy x_0 = x_init, the dynamics and SO(2) exactly;
    fc_k >= fc_min and |u| <= 1 are enforced by the local solver)."""
    from scipy.optimize import minimize
    from strom_inputs.models import pendulum_rollout

    pop = sdp.meta["pop"]
    N = pop.N
    meta = pop.meta
    p = meta["params"]
    th0, thd0 = meta["theta0"], meta["theta_dot0"]
    zbar = extract_raw(sdp, X)
    u0 = np.clip(np.array([zbar[5 * k + 4] for k in range(N)]), -1.0, 1.0)

    def J(u):
        return pop.objective(pendulum_rollout(N, u, th0, thd0, p))

    def fc_margin(u):
        z = pendulum_rollout(N, u, th0, thd0, p)
        fs = np.array([z[5 * k + 3] for k in range(1, N + 1)])
        return 1.0 - fs ** 2 - p.fc_min ** 2   # fc = sqrt(1 - fs^2) >= fc_min

    u = u0
    if refine:
        res = minimize(J, u0, method="SLSQP", bounds=[(-1.0, 1.0)] * N,
                       constraints=[{"type": "ineq", "fun": fc_margin}],
                       options={"maxiter": 300, "ftol": 1e-12})
        if res.success or np.all(fc_margin(res.x) >= -1e-12):
            u = np.clip(res.x, -1.0, 1.0)
    z_hat = pendulum_rollout(N, u, th0, thd0, p)
    feasible = bool(np.all(fc_margin(u) >= -1e-9))
    return z_hat, pop.objective(z_hat), feasible
