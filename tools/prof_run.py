"""Short run for ncu: `iters` sGS-ADMM iterations via the C-ABI on a bench config
(default pend30).  python tools/prof_run.py [config|N] [iters]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2406_05846_b200 as S
import bench
arg = sys.argv[1] if len(sys.argv) > 1 else "pend30"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg, N = (arg, None) if arg in bench.CONFIGS else ("pend30", int(arg))
torch.cuda.set_device(0)
st = torch.cuda.Stream()
sdp, _ = bench.make_sdp(cfg, N, 0)
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=1), stream=st)
g.iterate(iters)
st.synchronize()
print("done", g.residuals())
