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


# ---------------------------------------------------------------- KKT residuals (hand values)
def test_kkt_residuals_hand_values_1x1():
    """eq:strom:sgsadmm:kkt-residual at a constructed point of the 1x1 SDP
    min x s.t. x = 1: X = 3, y = 2, S = 0.5 gives, by hand,
    eta_p = |3 - 1| / (1 + 1) = 1, eta_d = |2 + 0.5 - 1| / (1 + 1) = 0.75,
    <C,X> = 3, <b,y> = 2, eta_g = |3 - 2| / (1 + 3 + 2) = 1/6."""
    from oracle import kkt_residuals
    ep, ed, eg, po, do = kkt_residuals(np.array([3.0]), np.array([1.0]), np.array([2.0]),
                                       np.array([0.5]), np.array([1.0]), np.array([3.0]),
                                       np.array([2.0]))
    assert (ep, ed, po, do) == (1.0, 0.75, 3.0, 2.0)
    assert abs(eg - 1.0 / 6.0) < 1e-16


def test_kkt_residuals_hand_values_2x2_offdiagonal():
    """Same residuals on a 2x2 block with off-diagonal entries, which fixes the norms as
    Frobenius norms of the matrices (svec with sqrt2 off-diagonal scaling, PAPER.md:571,
    reading Q15) and the '1 +' normalisations of PAPER.md:501-508. Row: tr X = 2.
    X = [[1, .5], [.5, 2]], y = .25, S = [[.5, .75], [.75, 1]], C = [[1, 1], [1, 0]]:
      A(X) - b = 3 - 2 = 1, eta_p = 1 / (1 + 2) = 1/3;
      A*y + S - C = [[-.25, -.25], [-.25, 1.25]], ||.||_F^2 = 3 * .0625 + 1.5625 = 1.75,
      ||C||_F^2 = 3, eta_d = sqrt(1.75) / (1 + sqrt(3));
      <C,X> = tr(CX) = 1 + 2 * .5 + 0 = 2, <b,y> = .5, eta_g = 1.5 / (1 + 2 + .5) = 3/7."""
    from oracle import kkt_residuals
    sdp = H.make_sdp([2], [{(0, 0, 0): 1.0, (0, 1, 1): 1.0}], [2.0], [np.array([[1.0, 1.0], [1.0, 0.0]])])
    o = Oracle(sdp)
    X = mat_to_svec(np.array([[1.0, 0.5], [0.5, 2.0]]))
    S = mat_to_svec(np.array([[0.5, 0.75], [0.75, 1.0]]))
    y = np.array([0.25])
    ep, ed, eg, po, do = kkt_residuals(o.apply_A(X), o.b, o.apply_At(y), S, o.C, X, y)
    assert abs(ep - 1.0 / 3.0) < 1e-15
    assert abs(ed - sqrt(1.75) / (1.0 + sqrt(3.0))) < 1e-15
    assert abs(po - 2.0) < 1e-15 and do == 0.5
    assert abs(eg - 3.0 / 7.0) < 1e-15


def test_kkt_residuals_vanish_at_closed_form_optimum():
    """At the exact primal-dual optimum of the 1x1 SDP (x = 1, y = 1, S = 0) every
    residual is zero; moving X alone changes eta_p and eta_g but not eta_d (eta_d
    involves only the dual pair)."""
    from oracle import kkt_residuals
    one = np.array([1.0])
    assert kkt_residuals(one, one, one, np.zeros(1), one, one, one) == (0.0, 0.0, 0.0, 1.0, 1.0)
    ep, ed, eg, _, _ = kkt_residuals(2 * one, one, one, np.zeros(1), one, 2 * one, one)
    assert ep > 0 and eg > 0 and ed == 0.0


# ---------------------------------------------------------------- sigma policy (reading Q2)
def test_sigma_rule_period_and_clamp_hand_sequence():
    """Reading Q2 (PAPER.md:454 only says sigma > 0): every `sigma_period` completed
    iterations, eta_d > ratio * eta_x -> sigma * factor; eta_x > ratio * eta_d ->
    sigma / factor; otherwise unchanged; clamped to [sigma_min, sigma_max]. Hand sequence
    (period 5, ratio 2, factor 1.5, clamp [0.5, 3])."""
    from oracle import sigma_update
    cfg = OracleConfig(sigma_period=5, sigma_ratio=2.0, sigma_factor=1.5, sigma_min=0.5, sigma_max=3.0)
    assert sigma_update(1.0, 4, 10.0, 1.0, cfg) == 1.0          # not a multiple of the period
    assert sigma_update(1.0, 5, 10.0, 1.0, cfg) == 1.5          # eta_d dominates: raise
    assert sigma_update(1.5, 10, 1.0, 10.0, cfg) == 1.0         # eta_x dominates: lower
    assert sigma_update(1.0, 15, 1.0, 1.9, cfg) == 1.0          # within the ratio band
    assert sigma_update(2.5, 20, 10.0, 1.0, cfg) == 3.0         # clamped above
    assert sigma_update(0.6, 25, 1.0, 10.0, cfg) == 0.5         # clamped below
    assert sigma_update(2.0, 25, 1.0, 10.0, OracleConfig(sigma_period=0)) == 2.0   # fixed sigma


def test_sigma_raises_dual_feasibility():
    """The premise of the rule's direction: sigma is the penalty on the dual constraint
    A*y + S = C (the augmented Lagrangian of PAPER.md:447-449), so a larger sigma makes
    that constraint's residual eta_d smaller and the primal-side residual eta_x larger."""
    sdp = compile_relaxation(models.pendulum(3, 0.3, 1.0))
    lo, hi = Oracle(sdp, OracleConfig(sigma=0.05)), Oracle(sdp, OracleConfig(sigma=20.0))
    lo.iterate(30); hi.iterate(30)
    assert hi.trace.eta_d[-1] < lo.trace.eta_d[-1] / 10
    assert hi.trace.eta_x[-1] > lo.trace.eta_x[-1]


def test_sigma_balancing_beats_fixed_and_reversed():
    """From a badly scaled sigma_0 the balancing rule reaches eta <= 1e-6 in fewer iterations
    than keeping sigma_0 fixed; the same rule with the direction reversed (factor < 1) does
    not converge at all. A sign error in the rule fails this test."""
    sdp = compile_relaxation(models.pendulum(3, 0.3, 1.0))
    pol = dict(sigma_period=10, sigma_ratio=1.5, sigma_factor=1.2)
    runs = {}
    for name, s0, kw, cap in (("policy_lo", 0.02, pol, 1500), ("fixed_lo", 0.02, {}, 1500),
                              ("reversed_lo", 0.02, dict(pol, sigma_factor=1 / 1.2), 1500),
                              ("policy_hi", 50.0, pol, 1500), ("fixed_hi", 50.0, {}, 1500)):
        o = Oracle(sdp, OracleConfig(sigma=s0, **kw))
        runs[name] = o.solve_to_tol(1e-6, cap)
    assert runs["policy_lo"][1] and not runs["fixed_lo"][1] and not runs["reversed_lo"][1], runs
    assert runs["policy_hi"][1] and runs["fixed_hi"][1] and runs["policy_hi"][0] < runs["fixed_hi"][0], runs
