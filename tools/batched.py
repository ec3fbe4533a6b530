"""Aggregate sGS-ADMM iters/s with B independent pendulum N=30 instances (states of the
paper's 10x10 grid) on one GPU: one handle + stream each, their iteration
graphs launched back to back (strom_admm_iterate is fully asynchronous), timed with events
on every stream (max over streams). NEXT-2 of SURVEY §8(f): the 30 moment blocks of one
instance occupy 30 of 148 SMs, a batch fills the rest.  python tools/batched.py [B ...]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
grid = models.pendulum_grid()
ITERS = 500
for B in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
    hs, sts = [], []
    for b in range(B):
        st = torch.cuda.Stream()
        sdp = compile_relaxation(models.pendulum(30, *grid[(b * 37 + 5) % 100]))
        hs.append(S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st))
        sts.append(st)
    for g in hs:
        g.iterate(200)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in hs]
    start = torch.cuda.Event(enable_timing=True)
    start.record(sts[0])
    for st in sts[1:]:
        st.wait_event(start)
    for (e0, _), st in zip(ev, sts):
        e0.record(st)
    for _ in range(ITERS // 100):
        for g in hs:
            g.iterate(100)
    for (_, e1), st in zip(ev, sts):
        e1.record(st)
    torch.cuda.synchronize()
    ms = max(start.elapsed_time(e1) for _, e1 in ev)
    print(json.dumps({"B": B, "iters_per_instance": ITERS, "ms": round(ms, 2),
                      "aggregate_iters_per_s": round(B * ITERS / (ms / 1e3), 1),
                      "per_instance_iters_per_s": round(ITERS / (ms / 1e3), 1)}), flush=True)
    del hs
