"""CPU tests of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/strom.h declares, validates inputs, and its host-side setup
factorisation of eps I + AA* solves the oracle's systems (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2406_05846_b200 as S
from paper_2406_05846_b200.build import build
from strom_inputs import compile_relaxation, models

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return S.load()


def test_header_symbols_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "strom.h")).read()
    declared = set(re.findall(r"\b(strom_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(S.EXPORTS), declared ^ set(S.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert "sm_100a" in S.strom_version()


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", S.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config(lib):
    cfg = S.strom_admm_default_config()
    assert cfg.sigma == 1.0 and 0 < cfg.tau < 2 and cfg.eps_rel == 1e-12


def _sdp(N=3):
    return compile_relaxation(models.pendulum(N, 0.3, 1.0))


def test_create_and_dims(lib):
    sdp = _sdp()
    h = S.StromSdp(sdp)
    assert h.dims() == (sdp.n, sdp.m, sdp.nblocks)


def _raw_create(nblocks, blocks, m, b):
    h = C.c_void_p()
    bb = np.ascontiguousarray(b, dtype=np.float64)
    return S.load().strom_sdp_create(C.byref(h), nblocks, blocks, m,
                                     bb.ctypes.data_as(C.POINTER(C.c_double)))


def _one_block(n=2, stage=0, rows=(0,), rowptr=(0, 1), col=(0,), val=(1.0,)):
    keep = [np.asarray(rows, np.int32), np.asarray(rowptr, np.int64), np.asarray(col, np.int32),
            np.asarray(val, np.float64), np.zeros(n * (n + 1) // 2)]
    blk = S.strom_block(n, stage, len(rows), keep[0].ctypes.data_as(C.POINTER(C.c_int32)),
                        keep[1].ctypes.data_as(C.POINTER(C.c_int64)),
                        keep[2].ctypes.data_as(C.POINTER(C.c_int32)),
                        keep[3].ctypes.data_as(C.POINTER(C.c_double)),
                        keep[4].ctypes.data_as(C.POINTER(C.c_double)))
    return blk, keep


def test_create_rejects_bad_input(lib):
    blk, keep = _one_block()
    arr = (S.strom_block * 1)(blk)
    assert _raw_create(1, arr, 1, [1.0]) == 0
    assert _raw_create(0, arr, 1, [1.0]) == -1                   # nblocks <= 0
    blk2, k2 = _one_block(col=(3,))                               # col >= svec(2) = 3
    assert _raw_create(1, (S.strom_block * 1)(blk2), 1, [1.0]) == -1
    assert "col out of range" in S.load().strom_last_error().decode()
    blk3, k3 = _one_block(rows=(1, 0), rowptr=(0, 1, 2), col=(0, 1), val=(1.0, 1.0))
    assert _raw_create(1, (S.strom_block * 1)(blk3), 2, [1.0, 0.0]) == -1   # rows not ascending
    # a row touching stages 0 and 2 is not a chain (Fig. 1 / PAPER.md:415)
    bA, kA = _one_block(n=1, stage=0, rows=(0,), rowptr=(0, 1), col=(0,))
    bB, kB = _one_block(n=1, stage=1, rows=(1,), rowptr=(0, 1), col=(0,))
    bC, kC = _one_block(n=1, stage=2, rows=(0,), rowptr=(0, 1), col=(0,))
    assert _raw_create(3, (S.strom_block * 3)(bA, bB, bC), 2, [1.0, 1.0]) == -1
    assert "not a chain" in S.load().strom_last_error().decode()


@pytest.mark.parametrize("case", ["pend3", "pend5", "synth", "toy"])
def test_host_factor_solve_matches_oracle(lib, case):
    from oracle import Oracle
    pop = {"pend3": models.pendulum(3, 0.3, 1.0), "pend5": models.pendulum(5, -0.2, 2.0),
           "synth": models.synthetic_shape("small", 4, seed=3), "toy": models.toy(3)}[case]
    sdp = compile_relaxation(pop)
    o = Oracle(sdp)
    h = S.StromSdp(sdp)
    rng = np.random.default_rng(0)
    for _ in range(2):
        r = o.A @ rng.standard_normal(o.n)
        y = h.host_solve(r)
        y2 = o.solve(r)
        # range quantities only: y is eps-amplified off range(A)
        assert np.linalg.norm(o.At @ (y - y2)) <= 1e-10 * np.linalg.norm(o.At @ y2)
        assert np.linalg.norm(o.K @ y - r) <= 1e-11 * np.linalg.norm(r)


def test_setup_without_gpu_fails_loudly(lib):
    """No CPU fallback: setup must refuse when no CUDA device is usable."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = S.StromSdp(_sdp())
    with pytest.raises(S.StromError):
        S.StromAdmm(h)


def test_setup_rejects_bad_config(lib):
    h = S.StromSdp(_sdp())
    for bad in ({"tau": 2.0}, {"sigma": 0.0}, {"check_every": 0}):
        cfg = S.strom_admm_default_config(**bad)
        with pytest.raises(S.StromError) as e:
            S.StromAdmm(h, cfg)
        assert e.value.status == -1


def test_handle_calls_validate_arguments(lib):
    """Entry points on a NULL handle return STROM_EINVAL (no GPU needed)."""
    import ctypes as C
    lam12 = (C.c_double * 4)()
    assert lib.strom_admm_extract(None, lam12, None) == -1
    assert lib.strom_admm_extract(None, None, None) == -1
    lb = C.c_double()
    assert lib.strom_admm_lower_bound(None, lam12, C.byref(lb), None) == -1
    assert lib.strom_admm_iterate(None, 1) == -1
