import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0); st = torch.cuda.Stream(); torch.cuda.set_stream(st)
sdp = compile_relaxation(models.pendulum(30, 0.1, 0.0))
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=50), stream=st)
prev = 0
for chunk in range(8):
    g.iterate(250); st.synchronize()
    v = g.residuals()["eig_sweeps"]; d = v - prev; prev = v
    tot, ge3, ge4 = d & ((1 << 24) - 1), (d >> 24) & ((1 << 20) - 1), d >> 44
    print(f"iters {chunk*250}-{chunk*250+250}: sweeps/block {tot/250/90:.2f}; 55-blocks with >=3 sweeps {ge3/250:.2f}/iter, >=4 {ge4/250:.2f}/iter")
