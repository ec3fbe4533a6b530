"""Data-driven warm start.

"we collect 60 x 120 solutions in the state space (theta, theta_dot) in [0, pi] x [-5, 5]
off-line. Given a new initial state (theta_0, theta_dot_0), we use Delaunay Triangulation to
search for three nearest neighbors among the solutions. A convex combination of these three
solutions is treated as the initial solution".

The paper's database holds MOSEK solutions; ours holds (X, y, S) from our own GPU solves
(`StromAdmm.get`), which is all the convex combination needs: every pendulum instance of one
horizon N has the same block sizes and constraint count (x_init only changes coefficients of
A and b, models.pendulum), so the stored iterates add entry by entry. The combination weights
are the barycentric coordinates of the query in the Delaunay simplex that contains it, i.e.
the three vertices of that triangle ("three nearest neighbors", reading Q-warm in DESIGN.md
§2). A query outside the convex hull of the database falls back to the three nearest
database points by Euclidean distance in the (scaled) state space, weighted by inverse
distance (still a convex combination).

Host-side logic only (numpy + scipy's Qhull triangulation); the result is handed to the GPU
path through `StromAdmm.set_start` / `set_start_device`.
"""
from __future__ import annotations

from typing import Optional, Sequence, Tuple

import numpy as np

__all__ = ["WarmStartDB"]


class WarmStartDB:
    """Database of solved states -> solutions, queried by Delaunay barycentric interpolation.

    `scale` rescales each state coordinate before triangulating and measuring distance
    (default: the bounding-box extent, so [0, pi] and [-5, 5] weigh equally); barycentric
    weights are invariant under this affine map, only the outside-hull fallback uses it.
    """

    def __init__(self, scale: Optional[Sequence[float]] = None):
        self.states: list = []
        self.sols: list = []
        self._scale = None if scale is None else np.asarray(scale, dtype=np.float64)
        self._tri = None

    def __len__(self) -> int:
        return len(self.states)

    def add(self, state: Sequence[float], X: np.ndarray, y: np.ndarray, S: np.ndarray):
        if self.sols:
            X0, y0, S0 = self.sols[0]
            if X.shape != X0.shape or y.shape != y0.shape or S.shape != S0.shape:
                raise ValueError("WarmStartDB.add: solution shapes differ from the database's "
                                 f"(X {X.shape} vs {X0.shape}, y {y.shape} vs {y0.shape})")
        self.states.append(np.asarray(state, dtype=np.float64).reshape(-1))
        self.sols.append((np.asarray(X, np.float64).copy(), np.asarray(y, np.float64).copy(),
                          np.asarray(S, np.float64).copy()))
        self._tri = None

    def _pts(self) -> Tuple[np.ndarray, np.ndarray]:
        P = np.stack(self.states)
        sc = self._scale
        if sc is None:
            ext = P.max(axis=0) - P.min(axis=0)
            sc = np.where(ext > 0, ext, 1.0)
        return P / sc, sc

    def weights(self, state: Sequence[float]) -> Tuple[np.ndarray, np.ndarray]:
        """(indices, weights) of the convex combination for `state`: weights >= 0, sum 1."""
        if len(self.states) == 0:
            raise ValueError("WarmStartDB.weights: empty database")
        q = np.asarray(state, dtype=np.float64).reshape(-1)
        P, sc = self._pts()
        qs = q / sc
        d = P.shape[1]
        if len(self.states) >= d + 1:
            if self._tri is None:
                from scipy.spatial import Delaunay
                try:
                    self._tri = Delaunay(P)
                except Exception:          # degenerate (collinear) database: no triangulation
                    self._tri = False
            if self._tri is not False:
                s = int(self._tri.find_simplex(qs[None, :])[0])
                if s >= 0:
                    T = self._tri.transform[s]                 # barycentric affine map
                    b = T[:d].dot(qs - T[d])
                    w = np.append(b, 1.0 - b.sum())
                    w = np.clip(w, 0.0, None)
                    return self._tri.simplices[s].copy(), w / w.sum()
        k = min(d + 1, len(self.states))
        dist = np.linalg.norm(P - qs[None, :], axis=1)
        idx = np.argsort(dist, kind="stable")[:k]
        if dist[idx[0]] == 0.0:
            return idx[:1], np.ones(1)
        w = 1.0 / dist[idx]
        return idx, w / w.sum()

    def query(self, state: Sequence[float]):
        """Convex combination (X, y, S) of the neighbours of `state`."""
        idx, w = self.weights(state)
        X = sum(wi * self.sols[i][0] for i, wi in zip(idx, w))
        y = sum(wi * self.sols[i][1] for i, wi in zip(idx, w))
        S = sum(wi * self.sols[i][2] for i, wi in zip(idx, w))
        return X, y, S

    def save(self, path: str):
        np.savez(path, states=np.stack(self.states),
                 X=np.stack([s[0] for s in self.sols]), y=np.stack([s[1] for s in self.sols]),
                 S=np.stack([s[2] for s in self.sols]),
                 scale=self._scale if self._scale is not None else np.zeros(0))

    @classmethod
    def load(cls, path: str) -> "WarmStartDB":
        z = np.load(path)
        db = cls(scale=z["scale"] if z["scale"].size else None)
        for st, X, y, S in zip(z["states"], z["X"], z["y"], z["S"]):
            db.add(st, X, y, S)
        return db
