"""Round-count study for the two-sided K-EIG (not product code): replays, in numpy, the
parallel (round-robin) two-sided Jacobi of eig2.cuh on B = V_prev^T X_b V_prev for the
X_b blocks the oracle produces along a pendulum run, and reports rounds per block until
every off-diagonal |b_ij| <= thr * ||X_b||_F (checked after every round, as the kernel's
barrier does), and the projection error against LAPACK.

    python tools/eig2_sim.py [N] [iters] [thr]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle, OracleConfig, svec_to_mat  # noqa: E402
from strom_inputs import compile_relaxation, models  # noqa: E402


def pairs_of_round(NP, r):
    def pos(j):
        if j == 0:
            return 0
        t = j - 1 + r
        if t >= NP - 1:
            t -= NP - 1
        return 1 + t
    return np.array([sorted((pos(P), pos(NP - 1 - P))) for P in range(NP // 2)])


NROT=[0,0]
def jacobi2(A, V0, thr_rel, max_rounds=4000):
    n = A.shape[0]
    NP = n + (n & 1)
    B = np.zeros((NP, NP)); V = np.zeros((NP, NP))
    B[:n, :n] = V0.T @ A @ V0
    V[:n, :n] = V0
    thr = thr_rel * np.linalg.norm(A)
    off = lambda M: np.abs(M - np.diag(np.diag(M))).max()
    if off(B) <= thr:
        return 0, B, V
    scheds = [pairs_of_round(NP, r) for r in range(NP - 1)]
    global NROT
    for k in range(max_rounds):
        pr = scheds[k % (NP - 1)]
        p, q = pr[:, 0], pr[:, 1]
        a, d, g = B[p, p], B[q, q], B[p, q]
        rot = np.abs(g) > thr
        NROT[0] += rot.sum(); NROT[1] += len(rot)
        dd = d - a
        g2 = 2 * g
        t = np.sign(dd + (dd == 0)) * g2 / (np.abs(dd) + np.sqrt(dd * dd + g2 * g2) + 1e-300)
        c = 1 / np.sqrt(1 + t * t)
        s = c * t
        c = np.where(rot, c, 1.0); s = np.where(rot, s, 0.0)
        J = np.eye(NP)
        J[p, p] = c; J[q, q] = c; J[p, q] = s; J[q, p] = -s
        B = J.T @ B @ J
        B[p, q] = 0.0; B[q, p] = 0.0
        V = V @ J
        if off(B) <= thr:
            return k + 1, B, V
    return max_rounds, B, V


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    thr_rel = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-15
    sdp = compile_relaxation(models.pendulum(N, 0.1, 0.0))
    o = Oracle(sdp, OracleConfig())
    rec = []
    orig = o.project

    def project(X):
        rec.append(X.copy())
        return orig(X)
    o.project = project
    o.iterate(iters)
    bo = np.asarray(sdp.block_offset)
    bn = np.asarray(sdp.block_n)
    big = [i for i in range(len(bn)) if bn[i] == bn.max()]
    Vw = {}
    for k in range(len(rec)):
        rounds, err = [], 0.0
        for i in big:
            A = svec_to_mat(rec[k][bo[i]:bo[i + 1]], bn[i])
            n = bn[i]
            V0 = Vw.get(i, np.eye(n))
            W, Q = np.linalg.eigh(A)
            P_ref = (Q * np.maximum(W, 0)) @ Q.T
            nr, B, V = jacobi2(A, V0, thr_rel)
            lam = np.diag(B)[:n]
            Vn = V[:n, :n]
            P = (Vn * np.maximum(lam, 0)) @ Vn.T
            err = max(err, np.abs(P - P_ref).max() / max(1.0, np.linalg.norm(A)))
            rounds.append(nr)
            Vw[i] = Vn            # the kernel keeps its own accumulated basis
        if k % 10 == 0 or k < 5:
            print(f"rotated frac {NROT[0]/max(1,NROT[1]):.2f}", end=' ')
            NROT[0]=NROT[1]=0
            print(f"iter {k:4d}: rounds mean {np.mean(rounds):6.1f} max {max(rounds):4d} "
                  f"(sweeps {max(rounds) / (n + (n & 1) - 1):.2f})  proj err {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
