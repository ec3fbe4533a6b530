"""A/B per-iteration time of two libstrom builds on pendulum N (alternating runs in
separate processes).  python tools/ab_time.py A B [N] [reps]; A and B are either built
libstrom.so files (same binding) or checkout directories (each with its own binding and
in-tree build, e.g. a git worktree of an older commit)."""
import os
import subprocess
import sys

A, B = sys.argv[1], sys.argv[2]
N = sys.argv[3] if len(sys.argv) > 3 else "30"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ.get("AB_ROOT", os.getcwd()))
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
N = int(sys.argv[1])
sdp = compile_relaxation(models.pendulum(N, 0.1, 0.0))
st = torch.cuda.Stream()
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st)
torch.cuda.set_stream(st)
g.iterate(300); st.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(st); g.iterate(1000); e1.record(st); st.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"{best:.3f}")
'''
res = {A: [], B: []}
for r in range(reps):
    for lib in (A, B):
        if os.path.isdir(lib):
            env = dict(os.environ, AB_ROOT=os.path.abspath(lib))
            env.pop("STROM_LIB", None)
        else:
            env = dict(os.environ, STROM_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", code, N], env=env, capture_output=True, text=True)
        try:
            res[lib].append(float(out.stdout.strip().splitlines()[-1]))
        except Exception:
            print(out.stdout, out.stderr)
            raise
for lib, v in res.items():
    print(f"{os.path.basename(lib):28s} us/iter " + " ".join(f"{x:.1f}" for x in v) + f"  best {min(v):.1f}")
