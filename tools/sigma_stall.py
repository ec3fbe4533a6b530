"""Sigma / tau study on stalled pendulum states (eta_g stall, DESIGN.md §9 item 3): fixed sigma
values and residual-balancing variants from a cold start, ITERS iterations each, final
residuals.  python tools/sigma_stall.py [iters]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
st = torch.cuda.Stream()
states = [(0.0, -0.555556), (0.1, 0.0), (0.0, 2.777778)]
variants = [dict(sigma=s) for s in (0.03, 0.1, 0.3, 1.0, 3.0, 10.0, 30.0)] + \
           [dict(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1),
            dict(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1, tau=1.0),
            dict(sigma=10.0, sigma_period=50, sigma_ratio=3.0, sigma_factor=1.2)]
for state in states:
    sdp = compile_relaxation(models.pendulum(30, *state))
    for v in variants:
        g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100, **v), stream=st)
        ok, it = g.solve(1e-6, iters)
        st.synchronize()
        r = g.residuals()
        print(json.dumps({"state": state, "variant": v, "ok": bool(ok), "iters": int(it),
                          "eta": [r["eta_p"], r["eta_d"], r["eta_g"]], "sigma": r["sigma"],
                          "pobj": r["pobj"], "dobj": r["dobj"], "iter_eta": r["iter_eta"]}), flush=True)
        del g
