"""K-EIG phase breakdown (profiling build, STROM_EIG_PROF): per-block clock64 stamps of
one launch after `iters` iterations of pendulum N.  python tools/eig_prof.py [N] [iters]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.path.join(ROOT, "tools", "ab", "libstrom_prof.so")
os.makedirs(os.path.dirname(lib), exist_ok=True)
os.environ["STROM_LIB"] = lib          # before the package import reads it
from paper_2406_05846_b200.build import build  # noqa: E402

if not os.path.exists(lib):
    build(force=True, out=lib, defines=("STROM_EIG_PROF",))
import paper_2406_05846_b200 as S  # noqa: E402
from strom_inputs import compile_relaxation, models  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
sdp = compile_relaxation(models.pendulum(N, 0.1, 0.0))
st = torch.cuda.Stream()
g = S.StromAdmm(S.StromSdp(sdp), S.strom_admm_default_config(check_every=1), stream=st)
raw = C.CDLL(lib)
nb = sdp.nblocks
bn = np.asarray(sdp.block_n)
names = ["gather", "warm U=AV", "sweeps", "eigpairs", "recon S", "store V"]
for it in (5, 50, iters, 3 * iters):
    g.iterate(it - g.residuals()["iter"] if it > g.residuals()["iter"] else 1)
    st.synchronize()
    buf = np.zeros((nb, 16), dtype=np.int64)
    assert raw.strom_debug_eig_prof(buf.ctypes.data_as(C.c_void_p), nb) == 0
    for n in sorted(set(bn.tolist()), reverse=True):
        sel = buf[bn == n]
        d = np.diff(sel[:, :7], axis=1)
        tot = sel[:, 6] - sel[:, 0]
        print(f"iter {it} n={n}: total cycles mean {tot.mean():.0f} max {tot.max()} | sweeps mean "
              f"{sel[:, 7].mean():.2f} max {sel[:, 7].max()} | per-sweep {(d[:, 2] / sel[:, 7]).mean():.0f}")
        print("    " + "  ".join(f"{nm} {d[:, k].mean():.0f}" for k, nm in enumerate(names)))
        if sel[:, 12:16].any():
            print("    eig2 round phases (thread 2, cycles per round): loads+2x2 %.0f  producer %.0f  stores+V %.0f  barrier %.0f" % tuple(
                (sel[:, 12 + k] / np.maximum(sel[:, 7], 1)).mean() for k in range(4)))
        if sel[:, 8].any():
            st0 = sel[:, 0]
            print("    detail (cycles from start): sched %.0f gather %.0f s %.0f staged %.0f Vcopy %.0f product %.0f" % tuple(
                (sel[:, k] - st0).mean() for k in (8, 9, 1, 10, 11, 2)))
