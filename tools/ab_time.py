"""A/B per-iteration time of two libstrom builds on pendulum N (alternating runs in
separate processes).  python tools/ab_time.py A B [N] [reps]; A and B are either built
libstrom.so files (same binding) or checkout directories (each with its own binding and
in-tree build, e.g. a git worktree of an older commit)."""
import os
import subprocess
import sys

# arguments: variants (a .so, a checkout directory, either with ",VAR=value" environment
# suffixes), then N and reps if numeric
variants = [a for a in sys.argv[1:] if "/" in a or a.endswith(".so")]
rest = [a for a in sys.argv[1:] if a not in variants]
N = rest[0] if rest else "30"           # pendulum horizon or a bench.py config name
reps = int(rest[1]) if len(rest) > 1 else 3
code = r'''
import os, sys, torch
sys.path.insert(0, os.environ.get("AB_ROOT", os.getcwd()))
import paper_2406_05846_b200 as S
from strom_inputs import compile_relaxation, models
arg = sys.argv[1]
if arg.isdigit():
    sdp = compile_relaxation(models.pendulum(int(arg), 0.1, 0.0))
else:                                  # a bench.py config name, e.g. carback30
    import bench
    sdp, _ = bench.make_sdp(arg, None, 0)
st = torch.cuda.Stream()
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=100), stream=st)
torch.cuda.set_stream(st)
warm, timed = (300, 1000) if arg.isdigit() else (20, 60)
g.iterate(warm); st.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(st); g.iterate(timed); e1.record(st); st.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1000.0 / timed)
print(f"{best:.3f}")
'''
res = {v: [] for v in variants}
for r in range(reps):
    for var in variants:
        lib, *envs = var.split(",")
        if os.path.isdir(lib):
            env = dict(os.environ, AB_ROOT=os.path.abspath(lib))
            env.pop("STROM_LIB", None)
        else:
            env = dict(os.environ, STROM_LIB=os.path.abspath(lib))
        env.update(dict(e.split("=", 1) for e in envs))
        out = subprocess.run([sys.executable, "-c", code, N], env=env, capture_output=True, text=True)
        try:
            res[var].append(float(out.stdout.strip().splitlines()[-1]))
        except Exception:
            print(out.stdout, out.stderr)
            raise
for var, v in res.items():
    print(f"{os.path.basename(var):36s} us/iter " + " ".join(f"{x:.1f}" for x in v) + f"  best {min(v):.1f}")
