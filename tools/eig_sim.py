"""Sweep-count study for K-EIG (not product code): replays the warm-started one-sided Jacobi
of eig.cuh in numpy on the X_b blocks the oracle produces along a pendulum run, and reports
per-block sweeps under the kernel's exit rules, with and without rotations between columns
of the same sign class (the projection needs only the +/- invariant subspaces).

    python tools/eig_sim.py [N] [iters]
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle, OracleConfig, svec_to_mat  # noqa: E402
from strom_inputs import compile_relaxation, models  # noqa: E402


def schedule(n):
    NP = n + (n & 1)
    rounds = []
    for r in range(NP - 1):
        def pos(j):
            if j == 0:
                return 0
            t = j - 1 + r
            if t >= NP - 1:
                t -= NP - 1
            return 1 + t
        pr = []
        for P in range(NP // 2):
            p, q = sorted((pos(P), pos(NP - 1 - P)))
            if q < n:
                pr.append((p, q))
        rounds.append(np.array(pr))
    return rounds


def jacobi(A, V0, cross_only=False, max_sweeps=40, mid_thr=1e-12, big_thr=1e-18):
    n = A.shape[0]
    s = 2.0 * np.linalg.norm(A)
    U = (A + s * np.eye(n)) @ V0
    tol2 = max(1e-15, 4 * n * 2.22e-16) ** 2
    sched = schedule(n)
    for sweep in range(max_sweeps):
        nrm = (U * U).sum(0)
        big = mid = rot = False
        big_corr = False
        for pr in sched:
            p, q = pr[:, 0], pr[:, 1]
            up, uq = U[:, p], U[:, q]
            ga = (up * uq).sum(0)
            al, be = nrm[p], nrm[q]
            ab = al * be
            sel = (ga * ga > tol2 * ab) & (ga != 0)
            if cross_only:
                lp, lq = np.sqrt(al) - s, np.sqrt(be) - s
                sel &= (np.sign(lp) != np.sign(lq))
            if not sel.any():
                continue
            rot = True
            big |= bool((ga[sel] ** 2 > big_thr * ab[sel]).any())
            big_corr |= bool((ga[sel] ** 2 > 1e-10 * ab[sel]).any())
            mid |= bool((ga[sel] ** 2 > mid_thr * ab[sel]).any())
            d = be - al
            g2 = 2 * ga
            t = np.sign(d + (d == 0)) * g2 / (np.abs(d) + np.sqrt(d * d + g2 * g2))
            c = 1 / np.sqrt(1 + t * t)
            sn = c * t
            c = np.where(sel, c, 1.0)
            sn = np.where(sel, sn, 0.0)
            nup = c * up - sn * uq
            nuq = sn * up + c * uq
            U[:, p], U[:, q] = nup, nuq
            nrm[p] = (nup * nup).sum(0)
            nrm[q] = (nuq * nuq).sum(0)
        if not rot or not big:
            return sweep + 1, U, s
        if CORR and not big_corr:
            # first-order simultaneous correction U <- U (I + Theta) from the Gram matrix
            G = U.T @ U
            nn = np.diag(G).copy()
            dn = np.sqrt(np.outer(nn, nn))
            cosm = np.abs(G) / dn
            np.fill_diagonal(cosm, 0.0)
            D = nn[None, :] - nn[:, None]          # D[p, q] = n_q - n_p
            with np.errstate(divide="ignore", invalid="ignore"):
                Th = np.where(cosm > 1e-12, G / D, 0.0)
            np.fill_diagonal(Th, 0.0)
            Th = np.triu(Th, 1)
            if np.all(np.isfinite(Th)) and np.abs(Th).max() <= 1e-6:
                Th = Th - Th.T
                U = U + U @ Th
                return sweep + 1.3, U, s
        if not mid:
            G = U.T @ U
            dn = np.sqrt(np.outer(np.diag(G), np.diag(G)))
            cosm = np.abs(G - np.diag(np.diag(G))) / dn
            if cross_only:
                lam = np.sqrt(np.diag(G)) - s
                cosm = np.where(np.sign(lam)[:, None] != np.sign(lam)[None, :], cosm, 0.0)
            if cosm.max() <= 1e-12:
                return sweep + 1, U, s
    return max_sweeps, U, s


def proj_from(U, s, A, cross_only):
    nr = np.linalg.norm(U, axis=0)
    lam = nr - s
    V = U / nr
    if not cross_only:
        return (V * np.maximum(lam, 0)) @ V.T, V
    Vp = V[:, lam > 0]
    Bp = Vp.T @ A @ Vp
    return Vp @ Bp @ Vp.T, V


MID = float(os.environ.get('MID', '1e-8'))
BIG = float(os.environ.get('BIG', '1e-18'))
CORR = os.environ.get('CORR', '0') == '1'
EVERY = os.environ.get('EVERY', '0') == '1'


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
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
        if (k % 25 and k < len(rec) - 5 and k > 5) and not (EVERY and k >= len(rec) - 50):
            # keep the warm basis current without recording
            for i in big:
                A = svec_to_mat(rec[k][bo[i]:bo[i + 1]], bn[i])
                Vw[i] = np.linalg.eigh(A)[1]
            continue
        sw = {False: [], True: []}
        err = 0.0
        for i in big:
            A = svec_to_mat(rec[k][bo[i]:bo[i + 1]], bn[i])
            V0 = Vw.get(i, np.eye(bn[i]))
            P_ref = (lambda W, Q: (Q * np.maximum(W, 0)) @ Q.T)(*np.linalg.eigh(A))
            for co, thr in ((False, 1e-12), (True, MID)):
                ns, U, s = jacobi(A, V0.copy(), False, mid_thr=thr, big_thr=(BIG if co else 1e-18))
                P, _ = proj_from(U, s, A, False)
                sw[co].append(ns)
                if co:
                    err = max(err, np.abs(P - P_ref).max() / max(1.0, np.abs(A).max()))
            Vw[i] = np.linalg.eigh(A)[1]
        print(f"iter {k:4d}: full sweeps mean {np.mean(sw[False]):.2f} max {max(sw[False])} | "
              f"mid={MID:g} big={BIG:g} mean {np.mean(sw[True]):.2f} max {max(sw[True])}  proj err {err:.1e}")


if __name__ == "__main__":
    main()
