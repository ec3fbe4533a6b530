"""Builds libstrom.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libstrom.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Compile csrc/ into `out`; `defines` (e.g. STROM_EIG_PROF) are for profiling builds."""
    OUT_ = out
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(HERE, "..", "include", "strom.h"))
    if not force and os.path.exists(OUT_):
        t = os.path.getmtime(OUT_)
        if all(os.path.getmtime(d) <= t for d in deps):
            return OUT_
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        cmd = [nvcc, "-c", s, "-o", o, "-O3", "-std=c++17", "-lineinfo", *ARCH,
               "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-v" if verbose else "-O3",
               "-I", os.path.join(HERE, "..", "include"), *["-D" + d for d in defines]]
        if s.endswith(".cpp"):
            cmd = [nvcc, "-x", "cu", *cmd[1:]] if False else cmd
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    cmd = [nvcc, "-shared", "-o", OUT_, *objs, *ARCH, "-Xcompiler", "-fopenmp", "-lgomp",
           "-lcusolver", "-lcublas", "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return OUT_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
