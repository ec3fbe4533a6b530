"""Setup time, device memory and iters/s for the paper's five problem shapes."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
torch.cuda.set_device(0)
st = torch.cuda.Stream()
cfgs = sys.argv[1:] or ["cartpole:30", "carback:30", "landing:50", "flying:60"]
for c in cfgs:
    shape, N = c.split(":"); N = int(N)
    t0 = time.time()
    pop = models.pendulum(N, 0.1, 0.0) if shape == "pendulum" else models.synthetic_shape(shape, N)
    sdp = compile_relaxation(pop)
    t1 = time.time()
    try:
        g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=10), stream=st)
    except Exception as e:
        print(json.dumps({"shape": c, "error": str(e)[:300]}), flush=True); continue
    t2 = time.time()
    g.iterate(20); st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); g.iterate(50); e1.record(st); st.synchronize()
    ms = e0.elapsed_time(e1) / 50
    kt = sorted(g.kernel_times(), key=lambda kv: -kv[1])[:6]
    print(json.dumps({"shape": c, "summary": sdp.summary(), "gen_s": round(t1 - t0, 1), "setup_s": round(t2 - t1, 1),
                      "factor": g.factor_info(), "ms_per_iter": ms, "iters_per_s": 1000 / ms,
                      "top_kernels_ms": kt, "res": g.residuals()}), flush=True)
    del g
