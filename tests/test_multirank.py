"""World-size-2 gloo tests (CPU) of the multi-GPU host logic of bench.py: every rank gets
its own problem instance (weak scaling over independent pendulum states of the paper's
grid) and timings are combined as the max over ranks."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    t = bench.max_over_ranks(1.0 + rank, ws)
    import paper_2406_05846_b200 as S
    nid = bench.share_nccl_id(S, rank)       # rank 0's NCCL id reaches every rank
    sdp, state = bench.make_sdp("pend5", None, rank)
    digest = float(np.sum(sdp.A_data * np.arange(sdp.nnz) % 7.0))
    q.put((rank, t, tuple(state), sdp.n, sdp.m, digest, nid))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_independent_instances_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, s0, n0, m0, d0, i0), (r1, t1, s1, n1, m1, d1, i1) = out
    assert len(i0) == 128 and i0 == i1 and any(i0)   # one NCCL id shared by all ranks
    assert t0 == t1 == 2.0                   # max over ranks
    assert s0 != s1                          # a different grid state per rank
    assert (n0, m0) == (n1, m1) == (8250, 8476)
    assert d0 != d1                          # different initial-condition rows -> different A
