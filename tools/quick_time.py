"""Scratch timing: per-iteration time of strom_admm_iterate on pendulum configs."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
for N in [int(x) for x in os.environ.get("QT_N", "5,30").split(",")]:
    t0 = time.time()
    sdp = compile_relaxation(models.pendulum(N, 0.1, 0.0))
    t1 = time.time()
    st = torch.cuda.Stream(); g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=50), stream=st); torch.cuda.set_stream(st)
    t2 = time.time()
    print(f"N={N} gen {t1-t0:.2f}s setup {t2-t1:.2f}s", g.factor_info(), "launches/iter", g.launches_per_iter(), flush=True)
    g.iterate(100); torch.cuda.synchronize()
    sw0 = g.residuals()["eig_sweeps"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.iterate(1000); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 1000
    r = g.residuals()
    print(f"N={N}: {ms*1000:.1f} us/iter, {1000/ms:.0f} iters/s, sweeps/block/iter {(r['eig_sweeps']-sw0)/1000/sdp.nblocks:.2f}", r, flush=True)
    print([(a, round(b*1000,1)) for a,b in g.kernel_times()], flush=True)
    if os.environ.get("QT_NOSOLVE"): continue
    ok, it = g.solve(1e-6, 100000 if N == 5 else 20000)
    torch.cuda.synchronize()
    print("solve", ok, it, g.residuals(), flush=True)
