"""Time to eta <= 1e-4 / 1e-5 / 1e-6 on the paper's other trajectory models (SURVEY.md §8(d)
C3-C5): one cold instance per model (seed 0 = the default start of
strom_inputs.paper_models, reading R-IS), the bench's sigma policy, strom_admm_solve in
graph launches of 100 iterations up to an iteration and wall-time budget; first crossings
tracked on the device. Generation and setup are timed separately. (The certificate's
extraction + local solve is pendulum-specific, so xi is not reported here.)

    python tools/time_to_tol_models.py [--out FILE] [config:max_iters ...]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--budget-s", type=float, default=90.0)
    ap.add_argument("cases", nargs="*", default=["cartpole30:20000", "carback30:20000", "landing50:10000",
                                                 "flying60:6000"])
    a = ap.parse_args()
    import torch
    import bench
    import paper_2406_05846_b200 as S
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    out = []
    for case in a.cases:
        cfg, maxit = case.split(":")
        maxit = int(maxit)
        t0 = time.perf_counter()
        sdp, state = bench.make_sdp(cfg, None, 0)
        t1 = time.perf_counter()
        g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100, **bench.SIGMA_POLICY),
                        stream=stream)
        stream.synchronize()
        t2 = time.perf_counter()
        it_done, ok, t_iter = 0, False, 0.0
        while it_done < maxit and t_iter < a.budget_s:
            t3 = time.perf_counter()
            ok, d = g.solve(1e-6, min(2000, maxit - it_done))
            stream.synchronize()
            t_iter += time.perf_counter() - t3
            it_done += d
            if ok:
                break
        r = g.residuals()
        row = {"config": cfg, "n": sdp.n, "m": sdp.m, "generate_s": t1 - t0, "setup_s": t2 - t1,
               "iterations": it_done, "iterate_s": t_iter, "us_per_iter": 1e6 * t_iter / max(it_done, 1),
               "reached_1e-6": bool(ok), "iter_eta": r["iter_eta"],
               "eta_final": [r["eta_p"], r["eta_d"], r["eta_g"]], "sigma_final": r["sigma"],
               "sigma_policy": bench.SIGMA_POLICY, "max_iters": maxit, "budget_s": a.budget_s}
        print(json.dumps(row), flush=True)
        out.append(row)
        del g
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
