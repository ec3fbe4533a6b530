"""Cold vs data-driven warm start on the pendulum grid.

The paper warm-starts from a 60 x 120 grid of MOSEK solutions; here the database is a coarser
grid of our own GPU solves (--db-theta x --db-dot states over [0, pi] x [-5, 5], each solved
to eta <= --tol cold), then every query state of the paper's 10 x 10 evaluation grid
(models.pendulum_grid) subsampled by --every is solved cold and warm (WarmStartDB.query ->
set_start) to the same tolerance. Reports iterations and wall seconds (setup + iterations)
per query and the medians. One GPU, one handle per instance.

  python tools/warm_grid.py --N 30 --db-theta 6 --db-dot 11 --every 7 --out gpurun_out/warm.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=30)
    ap.add_argument("--db-theta", type=int, default=6)
    ap.add_argument("--db-dot", type=int, default=11)
    ap.add_argument("--every", type=int, default=7)
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--maxiter", type=int, default=60000)
    ap.add_argument("--balance", action="store_true",
                    help="residual-balancing sigma policy of bench.py (reading R-new-2) instead of sigma = 1")
    ap.add_argument("--carry-sigma", action="store_true",
                    help="start the warm solve at the neighbours' converged sigma (weighted geometric mean)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch
    import paper_2406_05846_b200 as S
    from paper_2406_05846_b200.warmstart import WarmStartDB
    from strom_inputs import compile_relaxation, models
    stream = torch.cuda.Stream()
    pol = dict(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1) if a.balance else {}

    def solve(state, start=None, sigma=None):
        sdp = compile_relaxation(models.pendulum(a.N, *state))
        t0 = time.perf_counter()
        cfg = dict(pol, sigma=sigma) if sigma is not None else pol
        g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100, **cfg), stream=stream)
        if start is not None:
            g.set_start(*start)
        ok, it = g.solve(a.tol, a.maxiter)
        stream.synchronize()
        wall = time.perf_counter() - t0
        X, y, Sm, _ = g.get()
        r = g.residuals()
        return {"ok": bool(ok), "iters": int(it), "wall_s": wall, "sigma": r["sigma"],
                "eta": max(r["eta_p"], r["eta_d"], r["eta_g"])}, (X, y, Sm)

    db = WarmStartDB()
    sig = []
    t0 = time.perf_counter()
    for th in np.linspace(0.0, np.pi, a.db_theta):
        for thd in np.linspace(-5.0, 5.0, a.db_dot):
            res, sol = solve((float(th), float(thd)))
            db.add((th, thd), *sol)
            sig.append(res["sigma"])
    t_db = time.perf_counter() - t0

    rows = []
    for k, st in enumerate(models.pendulum_grid()):
        if k % a.every:
            continue
        cold, _ = solve(st)
        s0 = None
        if a.carry_sigma:
            idx, w = db.weights(st)
            s0 = float(np.exp(sum(wi * np.log(sig[i]) for i, wi in zip(idx, w))))
        warm, _ = solve(st, db.query(st), s0)
        rows.append({"state": list(st), "cold": cold, "warm": warm})
        print(json.dumps(rows[-1]), flush=True)

    def med(key, f):
        v = [r[key][f] for r in rows if r[key]["ok"]]
        return float(np.median(v)) if v else None
    out = {"N": a.N, "tol": a.tol, "sigma_policy": pol or "fixed sigma = 1", "carry_sigma": a.carry_sigma, "db_states": len(db), "db_build_s": t_db, "queries": len(rows),
           "cold_ok": sum(r["cold"]["ok"] for r in rows), "warm_ok": sum(r["warm"]["ok"] for r in rows),
           "median_iters": {"cold": med("cold", "iters"), "warm": med("warm", "iters")},
           "median_wall_s": {"cold": med("cold", "wall_s"), "warm": med("warm", "wall_s")},
           "rows": rows}
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
