"""Aggregate sGS-ADMM iters/s with B independent pendulum N=30 instances (grid states) on
one GPU, one handle + stream each, graphs launched back to back on their own streams."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
grid = models.pendulum_grid()
for B in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    hs, sts = [], []
    for b in range(B):
        st = torch.cuda.Stream()
        sdp = compile_relaxation(models.pendulum(30, *grid[(b * 37 + 5) % 100]))
        hs.append(S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st))
        sts.append(st)
    for g in hs: g.iterate(200)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rep in range(10):
        for g in hs: g.iterate(100)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"B": B, "aggregate_iters_per_s": B * 1000 / dt, "per_instance_iters_per_s": 1000 / dt}), flush=True)
    del hs
