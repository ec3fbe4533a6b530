"""Trajectory-optimisation POPs of the paper, built in rescaled coordinates.

* toy 1-D system (Example 1) -- the worked example whose
  moment/localizing/equality/consensus rows the paper prints;
* inverted pendulum (App. E.1) under reading R1
   which reproduces n = 49,500 and
  m = 47,351 at N = 30;
* a seeded synthetic chain with the same row families and
  the clique sizes of the larger models (car back-in |I| = 18 -> 190/19, flying
  robot |I| = 20 -> 231/21), used for throughput and scaling runs.

Rescaling (Q12): every variable lives in [-1, 1] (the pendulum
control u = u_max * u_hat); every constraint polynomial is later divided by its
max |coef| in `compile_relaxation`; the LQR loss (eq:exp:gen:lqr-loss,
PAPER.md:624-631) uses Q_x = Q_u = I in rescaled coordinates.
"""
from __future__ import annotations

from dataclasses import dataclass
from math import cos, sin, sqrt
from typing import List, Sequence, Tuple

import numpy as np

from .poly import Poly
from .relax import ChainPop


# ----------------------------------------------------------------------------
# Toy 1-D system
# ----------------------------------------------------------------------------
def toy(N: int = 3, dt: float = 0.1, Pf: float = 1.0, x_init: float = 2.0) -> ChainPop:
    """z = [x0; u0; x1; u1; ...; xN], I_k = (x_{k-1}, u_{k-1}, x_k).

    f_k = u_{k-1}^2 + x_{k-1}^2, f_N += Pf x_N^2; g_{k,1} = 1 - u_{k-1}^2;
    h_{k,1} = x_k + (dt - 1) x_{k-1} + dt u_{k-1} x_{k-1}; h_{1,2} = x_0 - x_init
    (eq:toy-as-sparse-pop).
    """
    cliques, f, g, h = [], [], [], []
    for k in range(1, N + 1):
        I = [2 * (k - 1), 2 * (k - 1) + 1, 2 * k]
        xp, u, x = (Poly.var(3, i) for i in range(3))
        fk = u * u + xp * xp
        if k == N:
            fk = fk + Pf * x * x
        hk = [x + (dt - 1.0) * xp + dt * (u * xp)]
        if k == 1:
            hk.append(xp - x_init)
        cliques.append(I); f.append(fk); g.append([1.0 - u * u]); h.append(hk)
    pop = ChainPop(d=2 * N + 1, cliques=cliques, f=f, g=g, h=h, R=[abs(x_init)] * N,
                   name=f"toy_N{N}")
    pop.meta = {"dt": dt, "Pf": Pf, "x_init": x_init, "gmax": [[1.0]] * N}
    return pop


def toy_rollout(N: int, u: Sequence[float], dt: float = 0.1, x_init: float = 2.0) -> np.ndarray:
    """Forward simulation x_k = x_{k-1} - dt (1 + u_{k-1}) x_{k-1}."""
    z = np.zeros(2 * N + 1)
    x = x_init
    for k in range(N):
        z[2 * k] = x
        z[2 * k + 1] = u[k]
        x = x - dt * (1.0 + u[k]) * x
    z[2 * N] = x
    return z


# ----------------------------------------------------------------------------
# Inverted pendulum (App. E.1), reading R1
# ----------------------------------------------------------------------------
@dataclass
class PendulumParams:
    m: float = 1.0
    l: float = 1.0
    b: float = 0.1
    g: float = 9.8
    dt: float = 0.1
    fc_min: float = 0.5
    u_max: float = 5.0
    Pf: float = 1.0


def pendulum_state(theta: float, theta_dot: float, dt: float) -> Tuple[float, float, float, float]:
    """x = (rc, rs, fc, fs) = (cos th, sin th, cos(th_dot dt), sin(th_dot dt)) (Q8, Q9)."""
    return (cos(theta), sin(theta), cos(theta_dot * dt), sin(theta_dot * dt))


def pendulum(N: int = 30, theta0: float = 0.1, theta_dot0: float = 0.0,
             p: PendulumParams | None = None) -> ChainPop:
    """Pendulum POP. Global z = [x_0, u_0, x_1, u_1, ..., x_N], x_k = (rc, rs, fc, fs),
    u_k = u_hat (u = u_max * u_hat). Clique k (1..N) = (x_{k-1}, u_{k-1}, x_k), |I| = 9.

    Per clique (R1): force balance (eq:exp:p:dis-dyn-constraints,
    PAPER.md:1116), rc/rs rotation updates, SO(2) of x_k
    (PAPER.md:1119-1120), SO(2) of x_{k-1} for k >= 2, and x_0 = x_init as four
    linear equalities in clique 1; inequalities fc_k >= fc_min (PAPER.md:1121,
    Q10) and u_max^2 - u_{k-1}^2 >= 0 -> 2N localizing blocks.
    """
    p = p or PendulumParams()
    x_init = pendulum_state(theta0, theta_dot0, p.dt)
    x_f = (-1.0, 0.0, 1.0, 0.0)  # theta = pi, theta_dot = 0
    nv = 9
    V = [Poly.var(nv, i) for i in range(nv)]
    rcp, rsp, fcp, fsp, u, rc, rs, fc, fs = V
    cliques, f, g, h = [], [], [], []
    for k in range(1, N + 1):
        I = [5 * (k - 1) + i for i in range(nv)]
        # LQR loss: (x_{k-1}-x_f)^T(x_{k-1}-x_f) + u_{k-1}^2 [+ Pf term]
        fk = u * u
        for j in range(4):
            fk = fk + (V[j] - x_f[j]) ** 2
        if k == N:
            for j in range(4):
                fk = fk + p.Pf * (V[5 + j] - x_f[j]) ** 2
        force = (p.m * p.l ** 2 / p.dt ** 2) * (fs - fsp) - p.u_max * u \
            + (p.m * p.g * p.l) * rsp + (p.b / p.dt) * fsp
        hk = [force,
              rc - (rcp * fcp - rsp * fsp),
              rs - (rsp * fcp + rcp * fsp),
              rc * rc + rs * rs - 1.0,
              fc * fc + fs * fs - 1.0]
        if k >= 2:
            hk += [rcp * rcp + rsp * rsp - 1.0, fcp * fcp + fsp * fsp - 1.0]
        else:
            hk += [V[j] - x_init[j] for j in range(4)]
        gk = [fc - p.fc_min, 1.0 - u * u]
        cliques.append(I); f.append(fk); g.append(gk); h.append(hk)
    pop = ChainPop(d=5 * N + 4, cliques=cliques, f=f, g=g, h=h, R=[1.0] * N,
                   name=f"pendulum_N{N}")
    pop.meta = {"params": p, "x_init": x_init, "x_f": x_f, "theta0": theta0,
                "theta_dot0": theta_dot0, "gmax": [[1.0 - p.fc_min, 1.0]] * N}
    return pop


def pendulum_rollout(N: int, u_hat: Sequence[float], theta0: float, theta_dot0: float,
                     p: PendulumParams | None = None) -> np.ndarray:
    """Forward simulation of the discretised pendulum."""
    p = p or PendulumParams()
    x = list(pendulum_state(theta0, theta_dot0, p.dt))
    z = np.zeros(5 * N + 4)
    for k in range(N):
        z[5 * k:5 * k + 4] = x
        z[5 * k + 4] = u_hat[k]
        rcp, rsp, fcp, fsp = x
        fs = fsp + (p.dt ** 2 / (p.m * p.l ** 2)) * (p.u_max * u_hat[k] - p.m * p.g * p.l * rsp
                                                      - (p.b / p.dt) * fsp)
        fc = sqrt(max(0.0, 1.0 - fs * fs))
        x = [rcp * fcp - rsp * fsp, rsp * fcp + rcp * fsp, fc, fs]
    z[5 * N:5 * N + 4] = x
    return z


def pendulum_grid(n_theta: int = 10, n_dot: int = 10) -> List[Tuple[float, float]]:
    """The 10x10 grid over [0, pi] x [-5, 5]."""
    return [(float(a), float(b)) for a in np.linspace(0.0, np.pi, n_theta)
            for b in np.linspace(-5.0, 5.0, n_dot)]


# ----------------------------------------------------------------------------
# Synthetic chain
# ----------------------------------------------------------------------------
SYNTH_SHAPES = {
    # name: (d_x, d_u, localizing blocks per clique) -- Table 1 d_x/d_u
    "carback": (7, 4, 22),     # |I| = 18 -> 190 / 19 (PAPER.md:702, 659 localizing at N=30)
    "landing": (8, 2, 10),     # |I| = 18 -> 190 / 19 (PAPER.md:704, 499 at N=50)
    "flying": (8, 4, 11),      # |I| = 20 -> 231 / 21 (PAPER.md:706, 659 at N=60)
    "small": (2, 1, 2),        # |I| = 5 -> 21 / 6, fast parity case
    "wide190": (2, 14, 2),     # |I| = 18 -> 190 / 19 blocks, few rows: parity of large K-EIG
    "wide231": (2, 16, 2),     # |I| = 20 -> 231 / 21 blocks
    "cartpole": (5, 3, 9),     # |I| = 13 -> 105 / 14 (273 localizing at N=30)
}


def synthetic_chain(N: int, dx: int, du: int, n_ineq: int, seed: int = 0,
                    name: str | None = None) -> ChainPop:
    """Random chain POP with the structure of eq:intro:trajopt:
    clique k = (x_{k-1}, u_{k-1}, x_k); dynamics x_k = A x_{k-1} + B u_{k-1} +
    bilinear(x_{k-1}, u_{k-1}) (degree 2), x_0 = x_init, box inequalities
    1 - z_j^2 >= 0 on n_ineq clique variables, LQR loss. Coefficients are seeded
    and scaled so rollouts from |x_init| <= 0.5 stay in [-1, 1] for short horizons.
    """
    rng = np.random.default_rng(seed)
    nv = 2 * dx + du
    V = [Poly.var(nv, i) for i in range(nv)]
    xp, uu, xx = V[:dx], V[dx:dx + du], V[dx + du:]
    Adyn = 0.9 * np.eye(dx) + 0.05 * rng.standard_normal((dx, dx))
    Bdyn = 0.1 * rng.standard_normal((dx, du))
    Cbil = 0.05 * rng.standard_normal((dx, dx, du))
    x_init = 0.5 * rng.uniform(-1.0, 1.0, dx)
    x_f = np.zeros(dx)
    cliques, f, g, h = [], [], [], []
    for k in range(1, N + 1):
        I = [(dx + du) * (k - 1) + i for i in range(nv)]
        fk = Poly.const(nv, 0.0)
        for j in range(dx):
            fk = fk + (xp[j] - x_f[j]) ** 2
        for j in range(du):
            fk = fk + uu[j] * uu[j]
        if k == N:
            for j in range(dx):
                fk = fk + (xx[j] - x_f[j]) ** 2
        hk = []
        for i in range(dx):
            e = xx[i] * 1.0
            for j in range(dx):
                e = e - float(Adyn[i, j]) * xp[j]
            for j in range(du):
                e = e - float(Bdyn[i, j]) * uu[j]
                for a in range(dx):
                    e = e - float(Cbil[i, a, j]) * (xp[a] * uu[j])
            hk.append(e)
        if k == 1:
            hk += [xp[j] - float(x_init[j]) for j in range(dx)]
        box_vars = list(range(dx, dx + du)) + list(range(dx + du, nv)) + list(range(dx))
        gk = [1.0 - V[box_vars[i % nv]] * V[box_vars[i % nv]] if i < nv
              else 1.0 - V[box_vars[i % nv]] * V[box_vars[(i + 1) % nv]] for i in range(n_ineq)]
        cliques.append(I); f.append(fk); g.append(gk); h.append(hk)
    pop = ChainPop(d=(dx + du) * N + dx, cliques=cliques, f=f, g=g, h=h, R=[1.0] * N,
                   name=name or f"synth_dx{dx}_du{du}_N{N}")
    gmax = [1.0 if i < nv else 2.0 for i in range(n_ineq)]
    pop.meta = {"x_init": x_init, "seed": seed, "gmax": [gmax] * N}
    return pop


def synthetic_shape(shape: str, N: int, seed: int = 0) -> ChainPop:
    dx, du, ni = SYNTH_SHAPES[shape]
    return synthetic_chain(N, dx, du, ni, seed=seed, name=f"synth_{shape}_N{N}")
