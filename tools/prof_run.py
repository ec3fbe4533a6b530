"""Short run for ncu: pendulum N (default 30), `iters` sGS-ADMM iterations via the C-ABI."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.cuda.set_device(0)
st = torch.cuda.Stream()
sdp = compile_relaxation(models.pendulum(N, 0.1, 0.0))
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=1), stream=st)
g.iterate(iters)
st.synchronize()
print("done", g.residuals())
