"""Data-driven warm start: Delaunay barycentric
combination of three database solutions. Pins: barycentric coordinates reproduce the query
point, affine fields are interpolated exactly (linear interpolation on a triangulation is
exact for affine functions), database points return their own solution, and a warm start from
neighbouring oracle solutions shortens the oracle's own solve."""
import numpy as np
import pytest

from paper_2406_05846_b200.warmstart import WarmStartDB


def _grid_db(field, nth=6, nd=7):
    db = WarmStartDB()
    for th in np.linspace(0.0, np.pi, nth):
        for thd in np.linspace(-5.0, 5.0, nd):
            X, y, S = field(np.array([th, thd]))
            db.add((th, thd), X, y, S)
    return db


def _affine(seed=0, n=9, m=5):
    rng = np.random.default_rng(seed)
    a = [rng.standard_normal(k) for k in (n, m, n)]
    B = [rng.standard_normal((k, 2)) for k in (n, m, n)]
    return lambda s: tuple(ai + Bi @ s for ai, Bi in zip(a, B))


def test_barycentric_weights_reproduce_query():
    db = _grid_db(_affine())
    rng = np.random.default_rng(1)
    for _ in range(200):
        q = np.array([rng.uniform(0, np.pi), rng.uniform(-5, 5)])
        idx, w = db.weights(q)
        assert len(idx) == 3 and np.all(w >= 0) and abs(w.sum() - 1) < 1e-14
        P = np.stack([db.states[i] for i in idx])
        assert np.allclose(w @ P, q, atol=1e-12)


def test_neighbours_are_corners_of_the_grid_cell():
    """On a regular grid the containing Delaunay triangle uses corners of the query's cell."""
    db = _grid_db(_affine())
    th, thd = np.linspace(0, np.pi, 6), np.linspace(-5, 5, 7)
    rng = np.random.default_rng(2)
    for _ in range(100):
        q = np.array([rng.uniform(0, np.pi), rng.uniform(-5, 5)])
        i, j = min(np.searchsorted(th, q[0]), 5), min(np.searchsorted(thd, q[1]), 6)
        cell = {(a, b) for a in (th[max(i - 1, 0)], th[i]) for b in (thd[max(j - 1, 0)], thd[j])}
        idx, w = db.weights(q)
        for k, wk in zip(idx, w):
            if wk > 1e-12:
                assert tuple(db.states[k]) in {tuple(map(float, c)) for c in cell}


def test_affine_fields_interpolated_exactly():
    f = _affine(3)
    db = _grid_db(f)
    rng = np.random.default_rng(4)
    for _ in range(50):
        q = np.array([rng.uniform(0, np.pi), rng.uniform(-5, 5)])
        for got, want in zip(db.query(q), f(q)):
            assert np.allclose(got, want, rtol=0, atol=1e-11)


def test_database_point_returns_its_solution():
    f = _affine(5)
    db = _grid_db(f)
    for k in (0, 10, 41):
        for got, want in zip(db.query(db.states[k]), db.sols[k]):
            assert np.allclose(got, want, atol=1e-12)


def test_outside_hull_and_small_databases():
    db = _grid_db(_affine())
    idx, w = db.weights((4.0, 7.0))                   # outside [0, pi] x [-5, 5]
    assert len(idx) == 3 and np.all(w > 0) and abs(w.sum() - 1) < 1e-14
    assert tuple(db.states[idx[0]]) == (np.pi, 5.0) and w[0] == w.max()
    one = WarmStartDB()
    one.add((0.0, 0.0), np.ones(3), np.ones(2), np.ones(3))
    X, y, S = one.query((1.0, 2.0))
    assert np.array_equal(X, np.ones(3))
    with pytest.raises(ValueError):
        one.add((1.0, 0.0), np.ones(4), np.ones(2), np.ones(3))
    with pytest.raises(ValueError):
        WarmStartDB().weights((0.0, 0.0))


def test_save_load_roundtrip(tmp_path):
    db = _grid_db(_affine(), 3, 3)
    p = str(tmp_path / "db.npz")
    db.save(p)
    db2 = WarmStartDB.load(p)
    q = (1.0, 0.5)
    for a, b in zip(db.query(q), db2.query(q)):
        assert np.array_equal(a, b)


def test_warm_start_shortens_oracle_solve():
    """Solutions at the three corners of a small triangle around the query warm-start the
    oracle's solve at the query: fewer iterations to eta <= 1e-5 than the cold start."""
    from oracle import Oracle
    from strom_inputs import compile_relaxation, models
    N, q = 3, (0.6, 1.0)
    db = WarmStartDB()
    for st in ((0.5, 0.8), (0.75, 1.0), (0.55, 1.3)):
        o = Oracle(compile_relaxation(models.pendulum(N, *st)))
        _, ok = o.solve_to_tol(1e-6, 20000)
        assert ok
        db.add(st, o.X, o.y, o.S)
    sdp = compile_relaxation(models.pendulum(N, *q))
    cold = Oracle(sdp)
    it_cold, ok_c = cold.solve_to_tol(1e-5, 20000)
    warm = Oracle(sdp)
    warm.set_start(*db.query(q))
    it_warm, ok_w = warm.solve_to_tol(1e-5, 20000)
    assert ok_c and ok_w and it_warm < it_cold, (it_warm, it_cold)
