"""Pins for the oracle (oracle/) against what the paper and mathematics fix.

Nothing here re-types the oracle's formulas: each test checks it against an
independent fact -- a closed-form optimum, an invariant of Algorithm 1, a
different library algorithm, or brute force on a tiny POP.
"""
from math import sqrt

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import (Oracle, OracleConfig, lower_bound, mat_to_svec, project_psd_block,
                    suboptimality_gap, svec_to_mat)
from strom_inputs import compile_relaxation, lift_rank1, models
from tests import sdp_helpers as H


def _sym(rng, n):
    G = rng.standard_normal((n, n))
    return (G + G.T) / 2


# ---------------------------------------------------------------- svec
def test_svec_roundtrip_and_inner_product():
    rng = np.random.default_rng(0)
    for n in (1, 2, 5, 10, 55):
        A, B = _sym(rng, n), _sym(rng, n)
        assert np.allclose(svec_to_mat(mat_to_svec(A), n), A, rtol=4e-16, atol=0)
        # <A, B> = tr(AB) = svec(A).svec(B) (SDPT3 convention)
        assert abs(mat_to_svec(A) @ mat_to_svec(B) - np.trace(A @ B)) < 1e-10 * n


# ---------------------------------------------------------------- projection
@pytest.mark.parametrize("n", [1, 3, 10, 55])
def test_projection_laws(n):
    rng = np.random.default_rng(n)
    X = _sym(rng, n)
    P, Pm = project_psd_block(X), project_psd_block(-X)
    assert np.linalg.eigvalsh(P)[0] >= -1e-12 * np.abs(X).max()
    assert np.allclose(project_psd_block(P), P, atol=1e-12)          # idempotent
    assert np.allclose(X, P - Pm, atol=1e-12)                         # Moreau
    assert abs(np.sum(P * Pm)) < 1e-10                                # complementarity
    # independent algorithm: Pi(X) = (X + |X|)/2 with |X| = sqrtm(X^2) (Schur method)
    absX = np.real(sla.sqrtm(X @ X))
    assert np.allclose(P, (X + absX) / 2, atol=1e-8)
    # nearest PSD point (Higham 1988): no random PSD Y is closer
    d0 = np.linalg.norm(X - P)
    for _ in range(20):
        G = rng.standard_normal((n, n)); Y = G @ G.T / n
        assert np.linalg.norm(X - Y) >= d0 - 1e-12
        Y2 = P + 1e-3 * (G @ G.T) / n
        assert np.linalg.norm(X - Y2) >= d0 - 1e-12


# ---------------------------------------------------------------- linear solve
def test_solve_matches_dense_and_residual():
    sdp = compile_relaxation(models.pendulum(2, 0.5, 1.0))
    o = Oracle(sdp)
    rng = np.random.default_rng(1)
    Ad = o.A.toarray()
    K = o.eps * np.eye(o.m) + Ad @ Ad.T
    for _ in range(3):
        r = Ad @ rng.standard_normal(o.n)       # r in range(A), as in Algorithm 1
        y = o.solve(r)
        assert np.linalg.norm(K @ y - r) <= 1e-12 * np.linalg.norm(r) * 1e2
        yd = np.linalg.solve(K, r)
        # y is determined only up to the eps-amplified null component (F2):
        # compare range quantities A*y.
        assert np.linalg.norm(Ad.T @ (y - yd)) <= 1e-9 * np.linalg.norm(Ad.T @ yd)
    # eps reading Q3: 1e-12 * max diag(AA*)
    assert abs(o.eps - 1e-12 * np.max(np.sum(Ad * Ad, axis=1))) < 1e-20


# ---------------------------------------------------------------- iteration invariants
@pytest.mark.parametrize("tau,sigma", [(1.0, 1.0), (1.618, 0.7), (1.95, 3.0)])
def test_iteration_invariants(tau, sigma):
    """F3: A(X^{k+1}) - b = (1-tau)(A(X^k) - b) - tau sigma eps y^{k+1};
    S^{k+1} in Omega+; <Pi(X_b), S^{k+1}> = 0; adjointness <A X, y> = <X, A* y>."""
    sdp = compile_relaxation(models.pendulum(3, 0.4, -1.0))
    o = Oracle(sdp, OracleConfig(sigma=sigma, tau=tau))
    rng = np.random.default_rng(2)
    o.set_start(X=rng.standard_normal(o.n) * 0.1, S=None)
    bo = sdp.block_offset
    for k in range(6):
        AXk = o.apply_A(o.X)
        out = o.iterate_once()
        lhs = o.apply_A(out["X"]) - o.b
        rhs = (1 - tau) * (AXk - o.b) - tau * sigma * o.eps * out["y"]
        assert np.linalg.norm(lhs - rhs) <= 1e-9 * (1 + np.linalg.norm(AXk - o.b))
        S = out["S"]; PiXb = out["Xb"] + sigma * S
        for beta, nb in enumerate(sdp.block_n):
            Sb = svec_to_mat(S[bo[beta]:bo[beta + 1]], int(nb))
            assert np.linalg.eigvalsh(Sb)[0] >= -1e-10 * (1 + np.abs(Sb).max())
        assert abs(PiXb @ S) <= 1e-9 * (1 + np.linalg.norm(PiXb) * np.linalg.norm(S))
        yv = rng.standard_normal(o.m); Xv = rng.standard_normal(o.n)
        assert abs(o.apply_A(Xv) @ yv - Xv @ o.apply_At(yv)) < 1e-9 * np.linalg.norm(Xv) * np.linalg.norm(yv)


# ---------------------------------------------------------------- closed-form optima
@pytest.mark.parametrize("case", ["one", "simplex", "lovasz", "chain"])
def test_closed_form_sdps(case):
    sdp, opt = {"one": H.one_by_one, "simplex": H.trace_simplex,
                "lovasz": H.lovasz_c5, "chain": H.two_stage_chain}[case]()
    o = Oracle(sdp, OracleConfig(sigma=1.0, tau=1.618, eps_rel=1e-14))
    it, ok = o.solve_to_tol(1e-9, 20000)
    assert ok, (case, it, o.residuals())
    ep, ed, eg, pobj, dobj = o.residuals()
    assert abs(pobj - opt) <= 1e-7 * (1 + abs(opt)), (pobj, opt)
    assert abs(dobj - opt) <= 1e-7 * (1 + abs(opt)), (dobj, opt)


# ---------------------------------------------------------------- relaxation value
def _toy_grid_opt(N, n_grid=41):
    """Brute force over a control grid + local polish: an upper bound p_hat."""
    import itertools
    from scipy.optimize import minimize
    pop = models.toy(N=N)
    grid = np.linspace(-1, 1, n_grid)
    best = (np.inf, None)
    for u in itertools.product(grid, repeat=N):
        v = pop.objective(models.toy_rollout(N, u))
        if v < best[0]:
            best = (v, np.array(u))
    res = minimize(lambda u: pop.objective(models.toy_rollout(N, u)), best[1],
                   bounds=[(-1, 1)] * N, method="L-BFGS-B")
    return min(best[0], res.fun)


def test_toy_relaxation_is_tight_lower_bound():
    """Theorem 1: p*_kappa <= p*; the toy's second-order
    relaxation is tight, so the SDP optimum equals the brute-force optimum."""
    N = 3
    sdp = compile_relaxation(models.toy(N=N))
    o = Oracle(sdp, OracleConfig(sigma=1.0))
    it, ok = o.solve_to_tol(1e-8, 50000)
    assert ok
    p_hat = _toy_grid_opt(N)
    ep, ed, eg, pobj, dobj = o.residuals()
    assert dobj <= p_hat + 1e-6
    assert abs(pobj - p_hat) <= 1e-5 * (1 + abs(p_hat))


def test_lower_bound_sound_for_garbage_y():
    """LB(y) <= <C, X(z_hat)> for ANY y, z_hat a feasible rollout."""
    N = 3
    pop = models.pendulum(N, 0.9, 2.0)
    sdp = compile_relaxation(pop)
    o = Oracle(sdp)
    rng = np.random.default_rng(5)
    z = models.pendulum_rollout(N, rng.uniform(-0.2, 0.2, N), 0.9, 2.0)
    p_hat = pop.objective(z)
    for scale in (1e-3, 1e-1, 1.0, 10.0):
        y = rng.standard_normal(o.m) * scale
        LB, lam = lower_bound(sdp, y, o.apply_At(y))
        assert LB <= p_hat + 1e-9
        # trace bound R_beta >= tr X(z_hat)_beta (Theorem 2)
    Xz = lift_rank1(sdp, z)
    for beta, nb in enumerate(sdp.block_n):
        tr = np.trace(svec_to_mat(Xz[sdp.block_offset[beta]:sdp.block_offset[beta + 1]], int(nb)))
        assert tr <= sdp.R_beta[beta] + 1e-12


def test_pendulum_small_certified():
    """Pendulum N=3: solve to 1e-6, certificate xi < 1% (PAPER.md:685 claim)."""
    from oracle import extract_pendulum
    sdp = compile_relaxation(models.pendulum(3, 0.3, 1.0))
    o = Oracle(sdp, OracleConfig(sigma=1.0))
    it, ok = o.solve_to_tol(1e-6, 20000)
    assert ok
    LB, _ = lower_bound(sdp, o.y, o.apply_At(o.y))
    z_hat, p_hat, feas = extract_pendulum(sdp, o.X)
    assert feas
    xi = suboptimality_gap(p_hat, LB)
    assert -1e-9 <= xi < 1e-2


def test_relaxation_hierarchy_is_monotone():
    """Theorem 1: p*_1 <= p*_2 <= p* — the first-order relaxation
    (App. B variant, kappa = 1) bounds the second-order one from below, both below the
    brute-force optimum of the toy problem."""
    N = 3
    p = []
    for kappa in (1, 2):
        o = Oracle(compile_relaxation(models.toy(N=N), kappa=kappa), OracleConfig(sigma=1.0))
        it, ok = o.solve_to_tol(1e-8, 50000)
        assert ok, kappa
        p.append(o.residuals()[3])
    p_hat = _toy_grid_opt(N)
    assert p[0] <= p[1] + 1e-6 and p[1] <= p_hat + 1e-6, (p, p_hat)
