"""Setup cost of repeated handles in one process (the MPC pattern): pendulum
N (default 30) at several grid states; prints strom_admm_setup_times per handle.
    STROM_PROF_SETUP=1 python tools/setup_time.py [N] [count]"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 5
grid = models.pendulum_grid()
torch.cuda.set_device(0)
st = torch.cuda.Stream()
for k in range(cnt):
    t0 = time.perf_counter()
    sdp = compile_relaxation(models.pendulum(N, *grid[(k * 37 + 5) % 100]))
    t1 = time.perf_counter()
    g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st)
    st.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"k": k, "generate_ms": 1e3 * (t1 - t0), "setup_ms": 1e3 * (t2 - t1),
                      "phases_ms": {a: round(b, 1) for a, b in g.setup_times().items()}}), flush=True)
    del g
