"""Product-side certificate (host post-processing) against the
oracle's independent extraction on a solved pendulum instance."""
import numpy as np

from oracle import Oracle, extract_pendulum, lower_bound
from paper_2406_05846_b200 import certify
from strom_inputs import compile_relaxation, lift_rank1, models


def test_certificate_matches_oracle_extraction():
    sdp = compile_relaxation(models.pendulum(4, 0.3, 1.0))
    o = Oracle(sdp)
    it, ok = o.solve_to_tol(1e-6, 20000)
    assert ok
    p1, z1, f1 = certify.pendulum_upper_bound(sdp, o.X)
    z2, p2, f2 = extract_pendulum(sdp, o.X)
    assert f1 and f2 and abs(p1 - p2) <= 1e-8 * (1 + abs(p2))
    LB, _ = lower_bound(sdp, o.y, o.apply_At(o.y))
    xi = certify.suboptimality_gap(p1, LB)
    assert 0.0 <= xi < 1e-2
    # the rounded point is feasible: A(X(z_hat)) = b
    import scipy.sparse as sp
    A = sp.csr_matrix((sdp.A_data, sdp.A_indices, sdp.A_indptr), shape=(sdp.m, sdp.n))
    assert np.max(np.abs(A @ lift_rank1(sdp, z1) - sdp.b)) < 1e-10


def test_extract_zbar_recovers_rank_one_point():
    """For X = X(z) exactly rank one, extraction returns z (Theorem 1(iii))."""
    sdp = compile_relaxation(models.pendulum(3, 0.5, -1.0))
    rng = np.random.default_rng(0)
    z = models.pendulum_rollout(3, rng.uniform(-0.3, 0.3, 3), 0.5, -1.0)
    zbar = certify.extract_zbar(sdp, lift_rank1(sdp, z))
    assert np.allclose(zbar, z, atol=1e-10)


def test_upper_bound_against_brute_force():
    """An independent pin of the certificate: on pendulum N=3 the
    controls are searched exhaustively (41^3 grid over [-1, 1]^3, feasible rollouts only,
    then a local polish from the best grid point). The valid lower bound LB must not exceed
    the global optimum, and the extraction + local solve of certify must reach it."""
    from scipy.optimize import minimize
    N, th0, thd0 = 3, 0.3, 1.0
    sdp = compile_relaxation(models.pendulum(N, th0, thd0))
    pop, p = sdp.meta["pop"], sdp.meta["pop"].meta["params"]
    o = Oracle(sdp)
    it, ok = o.solve_to_tol(1e-6, 20000)
    assert ok
    LB, _ = lower_bound(sdp, o.y, o.apply_At(o.y))
    p_hat, z_hat, feas = certify.pendulum_upper_bound(sdp, o.X)
    assert feas

    def J(u):
        return pop.objective(models.pendulum_rollout(N, u, th0, thd0, p))

    def margin(u):
        z = models.pendulum_rollout(N, u, th0, thd0, p)
        return 1.0 - z[[5 * k + 3 for k in range(1, N + 1)]] ** 2 - p.fc_min ** 2

    g = np.linspace(-1.0, 1.0, 41)
    best, ubest = np.inf, None
    for a in g:
        for b in g:
            for c in g:
                u = np.array([a, b, c])
                if np.all(margin(u) >= 0.0):
                    v = J(u)
                    if v < best:
                        best, ubest = v, u
    res = minimize(J, ubest, method="SLSQP", bounds=[(-1.0, 1.0)] * N,
                   constraints=[{"type": "ineq", "fun": margin}], options={"ftol": 1e-14, "maxiter": 500})
    p_star = min(best, res.fun if np.all(margin(res.x) >= -1e-12) else np.inf)
    assert LB <= p_star + 1e-8 * (1 + abs(p_star)), (LB, p_star)
    assert p_hat <= p_star + 1e-6 * (1 + abs(p_star)), (p_hat, p_star)
    assert p_hat >= p_star - 1e-6 * (1 + abs(p_star)), (p_hat, p_star)
