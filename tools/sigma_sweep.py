"""Time-to-tolerance experiment: pendulum N=30 cold start, several sigma policies."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
st = torch.cuda.Stream()
th, thd = float(sys.argv[1]), float(sys.argv[2])
maxit = int(sys.argv[3])
sdp = compile_relaxation(models.pendulum(30, th, thd))
h = S.StromSdp(sdp)
configs = [dict(sigma=1.0), dict(sigma=1.0, sigma_period=50, sigma_ratio=2.0, sigma_factor=1.2),
           dict(sigma=1.0, sigma_period=100, sigma_ratio=5.0, sigma_factor=1.5),
           dict(sigma=0.3), dict(sigma=3.0), dict(sigma=1.0, tau=1.95),
           dict(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1)]
for c in configs:
    g = S.StromAdmm(h, S.strom_admm_default_config(check_every=100, **c), stream=st)
    t0 = time.time()
    marks = {}
    done = 0
    for tol in (1e-4, 1e-5, 1e-6):
        ok, it = g.solve(tol, maxit - done)
        done += it
        marks[tol] = done if ok else None
        if not ok:
            break
    r = g.residuals()
    print(json.dumps({"cfg": c, "iters_to": {str(k): v for k, v in marks.items()}, "t": time.time() - t0,
                      "eta": [r["eta_p"], r["eta_d"], r["eta_g"]], "sigma_end": r["sigma"], "pobj": r["pobj"]}), flush=True)
