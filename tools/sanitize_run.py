"""Short run of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): pendulum N=5 iterations through the graphs, solve-to-tolerance, lower bound,
extraction, a 190-order block (4-CTA cluster K-EIG), in-process virtual ranks (the
partitioned solve kernels) and a batch.  compute-sanitizer --tool X python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models

torch.cuda.set_device(0)
sdp = compile_relaxation(models.pendulum(5, 0.3, 1.0))
hs = S.StromSdp(sdp)
g = S.StromAdmm(hs, S.strom_admm_default_config(check_every=2))
g.iterate(3)
g.solve(1e-3, 20)
X, y, Sm, r = g.get()
g.lower_bound(np.asarray(sdp.R_beta))
g.extract()
g.debug_solve(np.ones(sdp.m))
w = compile_relaxation(models.synthetic_shape("wide190", 2, seed=2))
gw = S.StromAdmm(S.StromSdp(w), S.strom_admm_default_config(check_every=1))
gw.iterate(2)
gw.get()
ranks = [S.StromAdmm(hs, S.strom_admm_default_config(check_every=2), rank=q, nranks=2, virtual=True) for q in range(2)]
S.strom_debug_link_virtual(ranks, hs)
S.strom_debug_iterate_virtual(ranks, 2)
ranks[0].get()
b = [S.StromAdmm(S.StromSdp(compile_relaxation(models.pendulum(3, t, 0.5))), S.strom_admm_default_config(check_every=2))
     for t in (0.2, 0.9)]
B = S.StromBatch(b, iters_per_launch=2)
B.iterate(4)
print("sanitize run ok", r["iter"])
