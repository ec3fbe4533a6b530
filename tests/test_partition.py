"""Horizon partition of the chain: host logic on CPU.

The partitioned solve of (eps I + AA*) y = r -- every rank eliminates its own stages down
to the boundary separators, ONE sum over ranks of the boundary right-hand side, the
reduced boundary system solved redundantly, local back substitution -- executed by the
library's host path (strom_debug_host_part) for every rank, combined, and checked against
the unpartitioned factored solve and the oracle's SuperLU solve. The world-size-2 test
runs the two ranks as separate processes that exchange the partials through a gloo
all_reduce, as the NCCL path does on GPUs.
"""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2406_05846_b200 as S
from oracle import Oracle
from strom_inputs import compile_relaxation, models

_CASES = {"pend5": lambda: models.pendulum(5, 0.3, 1.0),
          "pend8": lambda: models.pendulum(8, 0.7, -1.0),
          "synth": lambda: models.synthetic_shape("small", 6, seed=1)}


def _combine(ys, m):
    """Each row from the rank(s) that hold it; boundary rows are held (identically) by the
    two ranks they couple."""
    y = np.zeros(m)
    for yq in ys:
        nz = yq != 0
        assert np.all((y[nz] == 0) | (np.abs(y[nz] - yq[nz]) <= 1e-14 * np.abs(yq[nz]).max())), "ranks disagree"
        y[nz] = yq[nz]
    return y


@pytest.mark.parametrize("name", sorted(_CASES))
def test_partitioned_solve_matches_factored_solve(name):
    sdp = compile_relaxation(_CASES[name]())
    h = S.StromSdp(sdp)
    o = Oracle(sdp)
    rng = np.random.default_rng(0)
    r = o.apply_A(rng.standard_normal(sdp.n))       # r in range(A), as in Algorithm 1
    y_ref = o.solve(r)
    P = int(np.max(sdp.block_stage)) + 1
    # R = 1 is the unpartitioned host solve (test_abi.py::test_host_factor_solve_matches_oracle);
    # two ranks and one rank per stage bracket the partitions (each host_part call refactors)
    for R in (sorted({2, P}) if name != "pend8" else (P,)):
        sends = [h.host_part(R, q, r) for q in range(R)]
        recv = np.sum(sends, axis=0)
        assert recv.size == (R - 1) * (70 if name.startswith("pend") else recv.size // max(R - 1, 1))
        y = _combine([h.host_part(R, q, r, recv) for q in range(R)], sdp.m)
        assert np.linalg.norm(o.K @ y - r) <= 1e-12 * np.linalg.norm(r), (name, R)
        # y is unique only up to the eps-amplified null part (F2): compare A*y
        assert np.linalg.norm(o.apply_At(y - y_ref)) <= 1e-10 * np.linalg.norm(o.apply_At(y_ref)), (name, R)


def test_partition_rejects_bad_rank_counts():
    sdp = compile_relaxation(models.pendulum(3, 0.3, 1.0))
    h = S.StromSdp(sdp)
    r = np.ones(sdp.m)
    with pytest.raises(S.StromError):
        h.host_part(4, 0, r)           # more ranks than stages
    with pytest.raises(S.StromError):
        h.host_part(2, 2, r)           # rank out of range


def sdp_A(sdp):
    import scipy.sparse as sp
    return sp.csr_matrix((sdp.A_data, sdp.A_indices, sdp.A_indptr), shape=(sdp.m, sdp.n))


def _worker(rank, ws, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sdp = compile_relaxation(models.pendulum(4, 0.4, 2.0))
    h = S.StromSdp(sdp)
    r = np.asarray(sdp_A(sdp) @ np.random.default_rng(3).standard_normal(sdp.n))
    send = torch.from_numpy(h.host_part(ws, rank, r))
    dist.all_reduce(send)                    # the one exchange per solve
    y = h.host_part(ws, rank, r, send.numpy())
    q.put((rank, y, r))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_gloo_partitioned_solve():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, q)) for rk in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sdp = compile_relaxation(models.pendulum(4, 0.4, 2.0))
    o = Oracle(sdp)
    r = out[0][2]
    y = _combine([out[0][1], out[1][1]], sdp.m)
    assert np.linalg.norm(o.K @ y - r) <= 1e-12 * np.linalg.norm(r)
    assert np.linalg.norm(o.apply_At(y - o.solve(r))) <= 1e-10 * np.linalg.norm(o.apply_At(o.solve(r)))
