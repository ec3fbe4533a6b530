import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch, paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0); st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sdp = compile_relaxation(models.pendulum(30, 0.1, 0.0))
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=1), stream=st)
prev = 0
for it in range(2000):
    g.iterate(1); st.synchronize()
    v = g.residuals()["eig_sweeps"]; d = v - prev; prev = v
    if it in (100, 300, 500, 1000, 1500, 1999):
        print(f"iter {it}: sweeps {d & 0xffffffffff}, first-order completions {d >> 40} (of 30 blocks)")
