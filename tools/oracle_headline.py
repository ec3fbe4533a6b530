"""The oracle (CPU fp64, oracle/) on the headline MPC start (theta0, theta_dot0) = (0.1, 0)
 at N = 30 with the bench's sigma policy (reading Q2), logging eta every
1,000 iterations: evidence whether the GPU's eta_g plateau on this instance is the
algorithm's (VERDICT r1 'do this' 4).  python tools/oracle_headline.py [iters] [tau]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle, OracleConfig
from strom_inputs import compile_relaxation, models
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 1.618
sdp = compile_relaxation(models.pendulum(30, 0.1, 0.0))
o = Oracle(sdp, OracleConfig(sigma=1.0, sigma_period=20, sigma_ratio=1.5, sigma_factor=1.1, tau=tau))
t0 = time.time()
for k in range(iters // 1000):
    o.iterate(1000)
    ep, ed, eg, po, do = o.residuals()
    print(json.dumps({"iter": o.it, "eta_p": ep, "eta_d": ed, "eta_g": eg, "pobj": po, "dobj": do,
                      "sigma": o.sigma, "wall_s": round(time.time() - t0, 1)}), flush=True)
