"""ctypes binding of the C++ relaxation generator (strom_inputs/csrc/gen.cpp, NEXT-3;
include/strom_gen.h). `compile_arrays(pop, kappa, gs, hs)` returns the BlockSdp arrays that
`relax.compile_relaxation` would build, byte for byte (tests/test_generator.py), computed
per clique in parallel in C++. Input side only: no sGS-ADMM arithmetic."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libstrom_gen.so")
SRC = os.path.join(_HERE, "csrc", "gen.cpp")
_lib = None


def build(force: bool = False) -> str:
    """g++ -O3 -fopenmp (no FP contraction: the sums must round like the Python reference)."""
    hdr = os.path.join(_HERE, "..", "include", "strom_gen.h")
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(SRC),
                                                                          os.path.getmtime(hdr)):
        return LIB
    cmd = ["g++", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c++17", "-ffp-contract=off", "-o", LIB, SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("libstrom_gen build failed:\n" + r.stderr)
    return LIB


class _Clique(C.Structure):
    _fields_ = [("nvars", C.c_int32), ("vars", C.POINTER(C.c_int32)),
                ("f_nterms", C.c_int32), ("f_exp", C.POINTER(C.c_uint8)), ("f_coef", C.POINTER(C.c_double)),
                ("ng", C.c_int32), ("g_nterms", C.POINTER(C.c_int32)), ("g_exp", C.POINTER(C.c_uint8)),
                ("g_coef", C.POINTER(C.c_double)),
                ("nh", C.c_int32), ("h_nterms", C.POINTER(C.c_int32)), ("h_exp", C.POINTER(C.c_uint8)),
                ("h_coef", C.POINTER(C.c_double))]


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        lib.strom_gen_compile.restype = C.c_int32
        lib.strom_gen_compile.argtypes = [C.c_int32, C.POINTER(_Clique), C.c_int32, C.POINTER(C.c_void_p)]
        lib.strom_gen_sizes.argtypes = [C.c_void_p] + [C.c_void_p] * 4
        lib.strom_gen_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 11
        lib.strom_gen_free.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


def available() -> bool:
    try:
        load()
        return True
    except Exception:
        return False


def _terms(polys, nv):
    nt = [len(p.terms) for p in polys]
    exps = [m for p in polys for m in p.terms.keys()]
    coefs = [c for p in polys for c in p.terms.values()]
    e = np.asarray(exps, dtype=np.uint8).reshape(-1, nv) if exps else np.zeros((0, nv), np.uint8)
    return (np.asarray(nt, dtype=np.int32), np.ascontiguousarray(e),
            np.ascontiguousarray(np.asarray(coefs, dtype=np.float64)))


def compile_arrays(pop, kappa: int, gs, hs):
    lib = load()
    N = pop.N
    arr = (_Clique * N)()
    keep = []
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    for k in range(N):
        nv = len(pop.cliques[k])
        vars_ = np.asarray(pop.cliques[k], dtype=np.int32)
        fn, fe, fc = _terms([pop.f[k]], nv)
        gn, ge, gc = _terms(gs[k], nv)
        hn, he, hc = _terms(hs[k], nv)
        keep += [vars_, fe, fc, gn, ge, gc, hn, he, hc]
        arr[k] = _Clique(nv, p(vars_, C.c_int32), int(fn[0]), p(fe, C.c_uint8), p(fc, C.c_double),
                         len(gs[k]), p(gn, C.c_int32), p(ge, C.c_uint8), p(gc, C.c_double),
                         len(hs[k]), p(hn, C.c_int32), p(he, C.c_uint8), p(hc, C.c_double))
    res = C.c_void_p()
    st = lib.strom_gen_compile(N, arr, kappa, C.byref(res))
    if st != 0:
        raise ValueError(f"strom_gen_compile failed ({st})")
    nb, n, m, nnz = C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
    lib.strom_gen_sizes(res, C.byref(nb), C.byref(n), C.byref(m), C.byref(nnz))
    nb, n, m, nnz = nb.value, n.value, m.value, nnz.value
    out = {"block_n": np.empty(nb, np.int32), "block_stage": np.empty(nb, np.int32),
           "block_kind": np.empty(nb, np.int8), "block_offset": np.empty(nb + 1, np.int64),
           "A_indptr": np.empty(m + 1, np.int64), "A_indices": np.empty(nnz, np.int32),
           "A_data": np.empty(nnz, np.float64), "b": np.empty(m, np.float64), "C": np.empty(n, np.float64),
           "row_family": np.empty(m, np.int8), "row_stage": np.empty(m, np.int32)}
    lib.strom_gen_copy(res, *[out[k].ctypes.data for k in ("block_n", "block_stage", "block_kind", "block_offset",
                                                           "A_indptr", "A_indices", "A_data", "b", "C",
                                                           "row_family", "row_stage")])
    lib.strom_gen_free(res)
    return out
