"""The paper's full pendulum experiment: all 100 states of the
10 x 10 grid over (theta0, theta_dot0) in [0, pi] x [-5, 5], N = 30, solved cold on ONE GPU
as one strom_batch (NEXT-2; a concurrent graph branch per instance, each instance stops at
its own first iteration with eta <= tol), then the certificate per instance (LB on the GPU,
extraction on the GPU, local solve on the host -> xi).

Reports per instance: iterations to eta <= 1e-4 / 1e-5 / 1e-6 (tracked on the device),
final eta, xi, and the batch wall times (generation, setup, iterations, certificate) -- and
the aggregate: fraction with eta <= 1e-6 and xi < 1%, fraction with xi < 1%, median
iterations. The paper: mean (median) 31.2 s (14.6 s) per state at tol 1e-4, maxiter 10,000,
"about 10%" hard states.

  python tools/grid_solve.py [--N 30] [--maxiter 20000] [--out gpurun_out/grid.json]
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
    ap.add_argument("--maxiter", type=int, default=20000)
    ap.add_argument("--K", type=int, default=50, help="iterations per batch graph launch")
    ap.add_argument("--states", type=int, default=100, help="first S states of the grid")
    ap.add_argument("--out", default=None)
    ap.add_argument("--variant", dest="variants", action="append", default=[],
                    help='extra policy as JSON, e.g. \'{"sigma": 1.0, "sigma_period": 0, "tau": 1.618}\' '
                         '(the same instances re-solved cold)')
    a = ap.parse_args()

    import torch
    import bench
    import paper_2406_05846_b200 as S
    from paper_2406_05846_b200 import certify
    from strom_inputs import compile_relaxation, models

    torch.cuda.set_device(0)
    grid = models.pendulum_grid()[:a.states]
    t0 = time.perf_counter()
    sdps = [compile_relaxation(models.pendulum(a.N, th, thd)) for th, thd in grid]
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    cfg = dict(check_every=a.K, **bench.SIGMA_POLICY)
    # stream=None: each handle creates its own CUDA stream (torch recycles a pool of 32)
    hs = [S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(**cfg), stream=None)
          for sdp in sdps]
    bs = torch.cuda.Stream()
    batch = S.StromBatch(hs, iters_per_launch=a.K, stream=bs)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0

    B = len(hs)
    variants = [dict(bench.SIGMA_POLICY, tau=1.618)]
    for v in a.variants:
        variants.append(json.loads(v))
    results = []
    for vi, var in enumerate(variants):
        if vi > 0:                                 # same instances, new policy, cold restart
            for g in hs:
                g.reconfigure(**var)
                g.set_start()
        results.append(run_variant(a, hs, sdps, grid, batch, var, certify, torch))
    base = results[0]
    base["wall_s"].update({"generate": t_gen, "setup": t_setup})
    base["wall_s"]["total"] = sum(base["wall_s"][k] for k in ("generate", "setup", "iterate", "certificate"))
    base["wall_s"]["per_state_amortised"] = base["wall_s"]["total"] / B
    out = dict(base, variants=[{k: v for k, v in r.items() if k != "instances"} for r in results[1:]],
               variant_instances=[r["instances"] for r in results[1:]])
    print(json.dumps({k: v for k, v in out.items() if k not in ("instances", "variant_instances")}))
    if a.out:
        with open(a.out, "w") as f:
            f.write(json.dumps(out) + "\n")


def run_variant(a, hs, sdps, grid, batch, var, certify, torch):
    B = len(hs)
    t1 = time.perf_counter()
    ok, total, conv = batch.solve(1e-6, a.maxiter)
    torch.cuda.synchronize()
    t_iter = time.perf_counter() - t1
    t0 = time.perf_counter()
    rows = []
    for i, (g, sdp, st) in enumerate(zip(hs, sdps, grid)):
        r = g.residuals()
        lb, _ = g.lower_bound(np.asarray(sdp.R_beta))
        X, _, _, _ = g.get(y=False, S=False)
        _, vtop = g.extract()
        p_hat, z_hat, feas = certify.pendulum_upper_bound(sdp, X, vtop=vtop)
        xi = certify.suboptimality_gap(p_hat, lb) if feas else float("inf")
        eta = max(r["eta_p"], r["eta_d"], r["eta_g"])
        rows.append({"state": [round(st[0], 6), round(st[1], 6)], "iters": int(total[i]),
                     "iters_to": r["iter_eta"], "eta": eta, "eta_g": r["eta_g"],
                     "xi": xi, "lb": lb, "p_hat": p_hat, "sigma": r["sigma"]})
    t_cert = time.perf_counter() - t0
    eta6 = np.array([r["iters_to"]["1e-6"] is not None for r in rows])
    xi1 = np.array([r["xi"] < 1e-2 for r in rows])
    it6 = [r["iters_to"]["1e-6"] for r in rows if r["iters_to"]["1e-6"] is not None]
    return {
        "N": a.N, "states": B, "maxiter": a.maxiter, "policy": var,
        "fraction_eta1e-6_and_xi1pct": float(np.mean(eta6 & xi1)),
        "fraction_xi_below_1pct": float(np.mean(xi1)),
        "fraction_eta_1e-4": float(np.mean([r["iters_to"]["1e-4"] is not None for r in rows])),
        "median_iters_to_1e-6_over_converged": float(np.median(it6)) if it6 else None,
        "median_iters_to_1e-4": float(np.median([r["iters_to"]["1e-4"] for r in rows
                                                 if r["iters_to"]["1e-4"] is not None])),
        "median_xi": float(np.median([r["xi"] for r in rows])),
        "wall_s": {"iterate": t_iter, "certificate": t_cert},
        "instances": rows,
    }


if __name__ == "__main__":
    main()
