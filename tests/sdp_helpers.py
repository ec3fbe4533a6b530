"""Tiny hand-built SDPs with closed-form optima (test helpers, no method arithmetic)."""
from math import sqrt
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp


def svec_pos(r, c):
    if r > c:
        r, c = c, r
    return c * (c + 1) // 2 + r


def make_sdp(block_n, rows, b, C):
    """rows: list of dict {(beta, r, c): matrix-entry coefficient a} meaning the
    constraint sum a * X_beta[r, c] (symmetric A_i with a at (r,c),(c,r) for r!=c
    counted once as <A_i, X> = sum over the pair). C: list of dense symmetric
    matrices. Returns an object duck-typed like strom_inputs.BlockSdp."""
    block_n = np.asarray(block_n, dtype=np.int32)
    off = np.zeros(len(block_n) + 1, dtype=np.int64)
    off[1:] = np.cumsum(block_n.astype(np.int64) * (block_n + 1) // 2)
    n = int(off[-1])
    data, ind, ptr = [], [], [0]
    for row in rows:
        ent = {}
        for (beta, r, c), a in row.items():
            s = int(off[beta]) + svec_pos(r, c)
            # <A_i, X> with A_i symmetric: entry (r,c) counted as a * X_rc;
            # X_rc = svec_s / sqrt2 off-diagonal
            ent[s] = ent.get(s, 0.0) + (a if r == c else a / sqrt(2.0))
        for s in sorted(ent):
            ind.append(s); data.append(ent[s])
        ptr.append(len(ind))
    Cs = np.zeros(n)
    for beta, Cb in enumerate(C):
        nb = int(block_n[beta])
        for cc in range(nb):
            for rr in range(cc + 1):
                Cs[int(off[beta]) + svec_pos(rr, cc)] = Cb[rr, cc] * (1.0 if rr == cc else sqrt(2.0))
    return SimpleNamespace(
        block_n=block_n, block_offset=off, block_stage=np.zeros(len(block_n), dtype=np.int32),
        block_kind=np.zeros(len(block_n), dtype=np.int8),
        A_indptr=np.asarray(ptr, dtype=np.int64), A_indices=np.asarray(ind, dtype=np.int32),
        A_data=np.asarray(data, dtype=np.float64), b=np.asarray(b, dtype=np.float64), C=Cs,
        R_beta=np.ones(len(block_n)), n=n, m=len(rows), nblocks=len(block_n))


def lovasz_c5():
    """theta(C5) = sqrt(5): max <J,X> s.t. tr X = 1, X_ij = 0 on the 5 cycle edges
    (Lovasz 1979). As a min problem: min <-J, X>, optimum -sqrt(5)."""
    n = 5
    rows = [{(0, i, i): 1.0 for i in range(n)}]
    for i in range(n):
        j = (i + 1) % n
        rows.append({(0, min(i, j), max(i, j)): 1.0})
    b = [1.0] + [0.0] * n
    return make_sdp([n], rows, b, [-np.ones((n, n))]), -sqrt(5.0)


def trace_simplex(seed=0, sizes=(3, 4, 2)):
    """min sum <C_b, X_b> s.t. sum tr X_b = 1, X >= 0  ->  min_b lambda_min(C_b)."""
    rng = np.random.default_rng(seed)
    Cs = []
    for nb in sizes:
        G = rng.standard_normal((nb, nb))
        Cs.append((G + G.T) / 2)
    rows = [{(beta, i, i): 1.0 for beta, nb in enumerate(sizes) for i in range(nb)}]
    opt = min(np.linalg.eigvalsh(Cb)[0] for Cb in Cs)
    return make_sdp(list(sizes), rows, [1.0], Cs), opt


def one_by_one():
    """min x s.t. x = 1, x >= 0 -> 1."""
    return make_sdp([1], [{(0, 0, 0): 1.0}], [1.0], [np.ones((1, 1))]), 1.0


def two_stage_chain():
    """Two 2x2 blocks X, Y (stages 0, 1) with one consensus row X11 = Y00 and
    X00 = 1, Y11 = 1, min X01 + Y01 ... -> hand-solved: X = [[1,a],[a,t]], Y = [[t,c],[c,1]],
    objective 2a + 2c with |a| <= sqrt(t), |c| <= sqrt(t); plus t <= 1/4 via
    tr-type row X11 + ... Use: min 2 X01 + 2 Y01 + X11 (linear in t) ->
    minimise -4 sqrt(t) + t -> t = 4, but cap t via Y11 + Y00 = 2 -> t = 1, a = c = -1:
    optimum -4 + 1 = -3."""
    rows = [
        {(0, 0, 0): 1.0},                         # X00 = 1
        {(0, 1, 1): 1.0, (1, 0, 0): -1.0},        # consensus X11 = Y00
        {(1, 1, 1): 1.0},                         # Y11 = 1
        {(1, 0, 0): 1.0, (1, 1, 1): 1.0},         # Y00 + Y11 = 2
    ]
    C = [np.array([[0.0, 1.0], [1.0, 1.0]]), np.array([[0.0, 1.0], [1.0, 0.0]])]
    sdp = make_sdp([2, 2], rows, [1.0, 0.0, 1.0, 2.0], C)
    sdp.block_stage = np.array([0, 1], dtype=np.int32)
    return sdp, -3.0
