"""Time to certified gap (xi < 1%) on pendulum N=30 (MPC start) for several sigma policies."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_05846_b200 as S
from paper_2406_05846_b200 import certify
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
st = torch.cuda.Stream()
th, thd = float(sys.argv[1]), float(sys.argv[2])
budget = float(sys.argv[3])
sdp = compile_relaxation(models.pendulum(30, th, thd))
h = S.StromSdp(sdp)
cfgs = [dict(sigma=1.0), dict(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1),
        dict(sigma=1.0, sigma_period=50, sigma_ratio=2.0, sigma_factor=1.2), dict(sigma=0.5), dict(sigma=2.0),
        dict(sigma=1.0, tau=1.9)]
for c in cfgs:
    g = S.StromAdmm(h, S.strom_admm_default_config(check_every=2000, **c), stream=st)
    t0 = time.time(); it = 0; u_prev = None; out = None
    while time.time() - t0 < budget:
        g.iterate(10000); st.synchronize(); it += 10000
        lb, _ = g.lower_bound(np.asarray(sdp.R_beta))
        X, _, _, r = g.get(y=False, S=False)
        p_hat, z, feas = certify.pendulum_upper_bound(sdp, X, u_start=u_prev)
        u_prev = certify.pendulum_controls(z, 30)
        xi = certify.suboptimality_gap(p_hat, lb)
        out = {"it": it, "xi": xi, "lb": lb, "p_hat": p_hat, "t": time.time() - t0,
               "eta": [r["eta_p"], r["eta_d"], r["eta_g"]], "sigma": r["sigma"]}
        if xi < 0.01:
            break
    print(json.dumps({"cfg": c, "state": [th, thd], **out}), flush=True)
