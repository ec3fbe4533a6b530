"""Aggregate sGS-ADMM iters/s with B independent pendulum N=30 instances (states of the
paper's 10x10 grid) on one GPU, NEXT-2 of SURVEY §8(f): the 30 moment blocks
of one instance occupy 30 of 148 SMs, a batch fills the rest.
  graph   : strom_batch (one CUDA graph, a concurrent branch per instance)
  streams : one handle + stream each, their own graphs launched back to back
Timed with CUDA events on the launching stream(s).  python tools/batched.py [B ...]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
grid = models.pendulum_grid()
ITERS = 500
N = int(os.environ.get("BATCH_N", "30"))
for B in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8, 16]:
    hs, sts = [], []
    for b in range(B):
        st = torch.cuda.Stream()
        sdp = compile_relaxation(models.pendulum(N, *grid[(b * 37 + 5) % 100]))
        hs.append(S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st))
        sts.append(st)
    out = {"B": B, "N": N, "iters_per_instance": ITERS}
    # graph mode
    bs = torch.cuda.Stream()
    bat = S.StromBatch(hs, iters_per_launch=100, stream=bs)
    bat.iterate(200)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(bs)
    bat.iterate(ITERS)
    e1.record(bs)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["graph_aggregate_iters_per_s"] = round(B * ITERS / (ms / 1e3), 1)
    del bat
    # separate streams
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in hs]
    start = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(sts[0])
    for st in sts[1:]:
        st.wait_event(start)
    for _ in range(ITERS // 100):
        for g in hs:
            g.iterate(100)
    for (_, e), st in zip(ev, sts):
        e.record(st)
    torch.cuda.synchronize()
    ms = max(start.elapsed_time(e) for _, e in ev)
    out["streams_aggregate_iters_per_s"] = round(B * ITERS / (ms / 1e3), 1)
    print(json.dumps(out), flush=True)
    del hs
