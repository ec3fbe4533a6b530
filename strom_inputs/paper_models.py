"""The paper's other four trajectory problems (App. E) as chain POPs.

Each model is written in the paper's variables and constraints and then rescaled
(reading Q12): every variable is mapped affinely from its box to [-1, 1]
(`_Box`), constraints are substituted in the rescaled variables (their coefficients are
divided by max |coef| in `compile_relaxation`), and the LQR loss (eq:exp:gen:lqr-loss,
PAPER.md:624-631) uses Q_x = Q_u = I in the rescaled coordinates.

Readings shared with the pendulum (reading R1, which reproduces the
pendulum's printed sizes exactly): clique k carries the dynamics linking its states, the
SO(2) constraints of its later state and, for k >= 2, again those of its earlier state;
clique 1 carries x_0 = x_init as linear equalities instead; inequality constraints are
placed on the clique's later state and its control. Per-model readings (R-CP, R-CB, R-VL,
R-FR) are in DESIGN.md §2; the printed sizes they do and do not reproduce are pinned in
tests/test_generator.py.
"""
from __future__ import annotations

from math import cos, pi, sin
from typing import List, Sequence, Tuple

from .poly import Poly
from .relax import ChainPop


class _Box:
    """Clique-local rescaled variables: slot i holds z_hat in [-1, 1] with the physical value
    c_i + s_i z_hat (box [lo_i, hi_i])."""

    def __init__(self, boxes: Sequence[Tuple[float, float]]):
        self.n = len(boxes)
        self.c = [(lo + hi) / 2.0 for lo, hi in boxes]
        self.s = [(hi - lo) / 2.0 for lo, hi in boxes]
        self.hat = [Poly.var(self.n, i) for i in range(self.n)]
        self.phys = [self.c[i] + self.s[i] * self.hat[i] for i in range(self.n)]

    def to_hat(self, i: int, value: float) -> float:
        return (value - self.c[i]) / self.s[i]


def _lqr(B: _Box, xs: Sequence[int], us: Sequence[int], x_f_phys: Sequence[float], weight: float = 1.0):
    """(x_hat - x_hat_f)^T (x_hat - x_hat_f) + u_hat^T u_hat in rescaled coordinates."""
    f = Poly.const(B.n, 0.0)
    for i, xf in zip(xs, x_f_phys):
        f = f + weight * (B.hat[i] - B.to_hat(i, xf)) ** 2
    for i in us:
        f = f + weight * B.hat[i] * B.hat[i]
    return f


def _rot_updates(P, rc0, rs0, fc0, fs0, rc1, rs1):
    """eq:exp:p:dis-dyn-constraints-rcupdate/-rsupdate."""
    return [P[rc1] - (P[rc0] * P[fc0] - P[rs0] * P[fs0]),
            P[rs1] - (P[rs0] * P[fc0] + P[rc0] * P[fs0])]


def _so2(P, c, s):
    """eq:exp:p:dis-dyn-constraints-so2-r/-f."""
    return P[c] * P[c] + P[s] * P[s] - 1.0


# ----------------------------------------------------------------------------------------
# Cart-pole (App. E.2)
# ----------------------------------------------------------------------------------------
def cartpole(N: int = 30, a0: float = 0.0, a_dot0: float = 0.0, theta0: float = 0.1,
             theta_dot0: float = 0.0, m1: float = 1.0, m2: float = 0.3, l: float = 0.5,
             g: float = 9.8, dt: float = 0.1, fc_min: float = 0.5, a_max: float = 1.0,
             u_max: float = 10.0, Pf: float = 1.0, a_f: float = 0.0) -> ChainPop:
    """x_k = [a, rc, rs, fc, fs], control u_k. The Lie-group variational
    integrator couples a and rs at k-1, k, k+1, so clique k (k = 1..N)
    is (x_{k-1}, x_k, u_k, a_{k+1}, rs_{k+1}): |I| = 13, the printed size(M) = 105
    (reading R-CP). Clique k carries both integrator equations at step k,
    the rotation update x_{k-1} -> x_k, SO(2) of x_k (and of x_{k-1} for k >= 2),
    fc_k >= fc_min, u_max^2 - u_k^2 >= 0, a_max^2 - a_k^2 >= 0; clique 1 pins x_0 and
    a_1 = a_0 + dt a_dot_0. Target: a = a_f, theta = pi, theta_dot = 0."""
    boxes = [(-a_max, a_max)] + [(-1.0, 1.0)] * 4          # x_{k-1}
    boxes += [(-a_max, a_max)] + [(-1.0, 1.0)] * 4         # x_k
    boxes += [(-u_max, u_max), (-a_max, a_max), (-1.0, 1.0)]   # u_k, a_{k+1}, rs_{k+1}
    B = _Box(boxes)
    P = B.phys
    ap, rcp, rsp, fcp, fsp, a, rc, rs, fc, fs, u, an, rsn = range(13)
    x_f = (a_f, -1.0, 0.0, 1.0, 0.0)
    x_init = (a0, cos(theta0), sin(theta0), cos(theta_dot0 * dt), sin(theta_dot0 * dt))
    cliques, f, gs, hs = [], [], [], []
    for k in range(1, N + 1):
        # global layout [x_0, (x_1, u_1), (x_2, u_2), ..., (x_N, u_N), a_{N+1}, rs_{N+1}]
        xo = lambda j: 0 if j == 0 else 5 + 6 * (j - 1)
        I = [xo(k - 1) + i for i in range(5)] + [xo(k) + i for i in range(5)] + [xo(k) + 5]
        I += [xo(k + 1), xo(k + 1) + 2] if k < N else [6 * N + 5, 6 * N + 6]
        dd = P[an] - 2.0 * P[a] + P[ap]                     # a_{k+1} - 2 a_k + a_{k-1}
        hk = [(m1 + m2) / dt * dd + (m2 * l / dt) * (P[rsn] - 2.0 * P[rs] + P[rsp]) - dt * P[u],
              (l / dt) * (P[fs] - P[fsp]) + (1.0 / dt) * dd * P[rc] + g * dt * P[rs]]
        hk += _rot_updates(P, rcp, rsp, fcp, fsp, rc, rs)
        hk += [_so2(P, rc, rs), _so2(P, fc, fs)]
        if k >= 2:
            hk += [_so2(P, rcp, rsp), _so2(P, fcp, fsp)]
        else:
            hk += [P[i] - x_init[i] for i in range(5)] + [P[a] - (a0 + dt * a_dot0)]
        gk = [P[fc] - fc_min, u_max ** 2 - P[u] * P[u], a_max ** 2 - P[a] * P[a]]
        fk = _lqr(B, range(5), [u], x_f)
        if k == N:
            fk = fk + _lqr(B, range(5, 10), [], x_f, Pf)
        cliques.append(I); f.append(fk); gs.append(gk); hs.append(hk)
    pop = ChainPop(d=6 * N + 7, cliques=cliques, f=f, g=gs, h=hs, R=[1.0] * N, name=f"cartpole_N{N}")
    pop.meta = {"model": "cartpole", "x_init": x_init, "x_f": x_f, "dt": dt}
    return pop


# ----------------------------------------------------------------------------------------
# Car back-in (App. E.5)
# ----------------------------------------------------------------------------------------
def _square(cx: float, cy: float, side: float):
    h = side / 2.0
    return [(cx + h, cy + h), (cx - h, cy + h), (cx - h, cy - h), (cx + h, cy - h)]


def carback(N: int = 30, x0: float = 2.0, y0: float = 4.0, theta0: float = 1.0,
            L: float = 6.0, W: float = 2.5, dt: float = 0.25, ry_max: float = 8.0,
            v_max: float = 4.0, w_max: float = 0.5, Pf: float = 10.0) -> ChainPop:
    """x_k = [x, y, rc, rs], u_k = [v, w, fc, fs] and the separating-line
    lifting (A1, B1, C1, A2, B2, C2)_k (eq:exp:cr:separation).
    Clique k (k = 0..N-1) = (x_k, u_k, ABC_k, x_{k+1}): |I| = 18, size(M) = 190.
    Per clique: position updates, the third-order fs(w) relation, rotation update x_k ->
    x_{k+1}, SO(2) of x_{k+1} and of the control pair (fc, fs) [and of x_k for k >= 1],
    the two unit spheres on (A, B, C); 16 separation inequalities (car vertices of x_k,
    eq:exp:cr:car-vertices, and obstacle vertices), rx_max^2 - x_{k+1}^2, ry_max^2 -
    y_{k+1}^2, v_max^2 - v_k^2, w_max^2 - w_k^2 >= 0 (reading R-CB). rx_max = |x0| + 2
    (the printed x0 + 2, reading Q23, made a valid box for x0 < 0). Obstacles: squares of
    side 8 at (+-6, -4); target (0, -3, pi/2)."""
    rx_max = abs(x0) + 2.0
    st = [(-rx_max, rx_max), (-ry_max, ry_max), (-1.0, 1.0), (-1.0, 1.0)]
    boxes = st + [(-v_max, v_max), (-w_max, w_max), (-1.0, 1.0), (-1.0, 1.0)] + [(-1.0, 1.0)] * 6 + st
    B = _Box(boxes)
    P = B.phys
    X, Y, RC, RS, V_, Wv, FC, FS = range(8)
    A1, B1, C1, A2, B2, C2 = range(8, 14)
    X1, Y1, RC1, RS1 = range(14, 18)
    x_f = (0.0, -3.0, cos(pi / 2), sin(pi / 2))
    x_init = (x0, y0, cos(theta0), sin(theta0))
    obst = [_square(6.0, -4.0, 8.0), _square(-6.0, -4.0, 8.0)]
    cliques, f, gs, hs = [], [], [], []
    for k in range(N):
        I = [14 * k + i for i in range(18)]
        hk = [P[X1] - P[X] - dt * P[V_] * P[RC],
              P[Y1] - P[Y] - dt * P[V_] * P[RS],
              P[FS] - (dt * P[Wv] - (dt * P[Wv]) ** 3 * (1.0 / 6.0))]
        hk += _rot_updates(P, RC, RS, FC, FS, RC1, RS1)
        hk += [_so2(P, RC1, RS1), _so2(P, FC, FS)]
        hk += [P[A1] * P[A1] + P[B1] * P[B1] + P[C1] * P[C1] - 1.0,
               P[A2] * P[A2] + P[B2] * P[B2] + P[C2] * P[C2] - 1.0]
        if k >= 1:
            hk += [_so2(P, RC, RS)]
        else:
            hk += [P[i] - x_init[i] for i in range(4)]
        # car vertices of x_k (eq:exp:cr:car-vertices)
        cx = [P[X] + (L / 2) * P[RC] * sx - (W / 2) * P[RS] * sy for sx, sy in ((1, 1), (-1, 1), (-1, -1), (1, -1))]
        cy = [P[Y] + (L / 2) * P[RS] * sx + (W / 2) * P[RC] * sy for sx, sy in ((1, 1), (-1, 1), (-1, -1), (1, -1))]
        gk = []
        for (Aa, Bb, Cc), ob in zip(((A1, B1, C1), (A2, B2, C2)), obst):
            gk += [P[Aa] * cx[i] + P[Bb] * cy[i] + P[Cc] for i in range(4)]
            gk += [-(P[Aa] * ox + P[Bb] * oy + P[Cc]) for ox, oy in ob]
        gk += [rx_max ** 2 - P[X1] * P[X1], ry_max ** 2 - P[Y1] * P[Y1],
               v_max ** 2 - P[V_] * P[V_], w_max ** 2 - P[Wv] * P[Wv]]
        fk = _lqr(B, range(4), [V_, Wv], x_f)
        if k == N - 1:
            fk = fk + _lqr(B, range(14, 18), [], x_f, Pf)
        cliques.append(I); f.append(fk); gs.append(gk); hs.append(hk)
    pop = ChainPop(d=14 * N + 4, cliques=cliques, f=f, g=gs, h=hs, R=[1.0] * N, name=f"carback_N{N}")
    pop.meta = {"model": "carback", "x_init": x_init, "x_f": x_f, "dt": dt}
    return pop


# ----------------------------------------------------------------------------------------
# Vehicle landing (App. E.3) and flying robot (App. E.4, 1667-1696)
# ----------------------------------------------------------------------------------------
def _planar(N, nu, x0, boxes_x, box_u, dyn, ineq_u, x_init, x_f, Pf, fc_min, name):
    """Shared layout of the two planar rigid-body models: x_k = [x, y, vx, vy, rc, rs, fc,
    fs], controls u_k (nu). Clique k (k = 0..N-1) = (x_k, u_k,
    x_{k+1}): |I| = 16 + nu. Per clique: `dyn` (the printed discrete dynamics), rotation
    update x_k -> x_{k+1}, SO(2) (r and f) of x_{k+1} [and of x_k for k >= 1];
    inequalities on u_k (`ineq_u`) and on x_{k+1}: the position / velocity boxes and
    fc_{k+1} >= fc_min."""
    boxes = list(boxes_x) + [box_u] * nu + list(boxes_x)
    B = _Box(boxes)
    P = B.phys
    nx = 8
    s1 = nx + nu
    cliques, f, gs, hs = [], [], [], []
    for k in range(N):
        I = [(nx + nu) * k + i for i in range(2 * nx + nu)]
        hk = dyn(P, nx, nu)
        hk += _rot_updates(P, 4, 5, 6, 7, s1 + 4, s1 + 5)
        hk += [_so2(P, s1 + 4, s1 + 5), _so2(P, s1 + 6, s1 + 7)]
        if k >= 1:
            hk += [_so2(P, 4, 5), _so2(P, 6, 7)]
        else:
            hk += [P[i] - x_init[i] for i in range(nx)]
        gk = ineq_u(P, nx, nu)
        for i, (lo, hi) in enumerate(boxes_x[:4]):
            gk.append((P[s1 + i] - lo) * (hi - P[s1 + i]))
        gk.append(P[s1 + 6] - fc_min)
        fk = _lqr(B, range(nx), range(nx, nx + nu), x_f)
        if k == N - 1:
            fk = fk + _lqr(B, range(s1, s1 + nx), [], x_f, Pf)
        cliques.append(I); f.append(fk); gs.append(gk); hs.append(hk)
    pop = ChainPop(d=(nx + nu) * N + nx, cliques=cliques, f=f, g=gs, h=hs, R=[1.0] * N, name=f"{name}_N{N}")
    pop.meta = {"model": name, "x_init": x_init, "x_f": x_f}
    return pop


def _state(x, y, vx, vy, th, thd, dt):
    return (x, y, vx, vy, cos(th), sin(th), cos(thd * dt), sin(thd * dt))


def landing(N: int = 50, x0: float = 20.0, y0: float = 80.0, vx0: float = 0.0, vy0: float = 0.0,
            theta0: float = 0.1, theta_dot0: float = 0.0, m: float = 1.0, Iz: float = 50.0, L: float = 5.0,
            g: float = 9.8, dt: float = 0.2, fc_min: float = 0.7, rx_max: float = 100.0, ry_min: float = 10.0,
            ry_max: float = 120.0, v_max: float = 20.0, u_max: float = 8.0, Pf: float = 10.0) -> ChainPop:
    """Vehicle landing: m (v_{k+1} - v_k) = dt (u1 + u2) (-rs, rc) - dt m g
    (the printed '- m g' read with the step dt, reading R-VL), I (fs_{k+1} - fs_k) =
    L dt^2 (u2 - u1), u_i (u_max - u_i) >= 0. Target x = 0, y = 10, theta = 0, at rest."""
    def dyn(P, nx, nu):
        s1 = nx + nu
        u1, u2 = P[nx], P[nx + 1]
        return [P[s1] - P[0] - dt * P[2], P[s1 + 1] - P[1] - dt * P[3],
                m * (P[s1 + 2] - P[2]) + dt * (u1 + u2) * P[5],
                m * (P[s1 + 3] - P[3]) - dt * (u1 + u2) * P[4] + dt * m * g,
                Iz * (P[s1 + 7] - P[7]) - L * dt * dt * (u2 - u1)]
    bx = [(-rx_max, rx_max), (ry_min, ry_max), (-v_max, v_max), (-v_max, v_max)] + [(-1.0, 1.0)] * 4
    return _planar(N, 2, None, bx, (0.0, u_max), dyn,
                   lambda P, nx, nu: [P[nx + i] * (u_max - P[nx + i]) for i in range(nu)],
                   _state(x0, y0, vx0, vy0, theta0, theta_dot0, dt), _state(0.0, 10.0, 0.0, 0.0, 0.0, 0.0, dt),
                   Pf, fc_min, "landing")


def flying(N: int = 60, x0: float = 5.0, y0: float = 5.0, vx0: float = 0.0, vy0: float = 0.0,
           theta0: float = 0.5, theta_dot0: float = 0.0, alpha: float = 0.2, beta: float = 0.2,
           dt: float = 0.2, fc_min: float = 0.7, rx_max: float = 10.0, ry_max: float = 10.0,
           v_max: float = 10.0, u_max: float = 8.0, Pf: float = 10.0) -> ChainPop:
    """Flying robot: v_{k+1} - v_k = dt (u1 - u2 + u3 - u4) (rc, rs),
    fs_{k+1} - fs_k = dt^2 alpha (u2 - u1) + dt^2 beta (u3 - u4), u_i (u_max - u_i) >= 0.
    Target: the origin at rest with theta = 0."""
    def dyn(P, nx, nu):
        s1 = nx + nu
        T = P[nx] - P[nx + 1] + P[nx + 2] - P[nx + 3]
        return [P[s1] - P[0] - dt * P[2], P[s1 + 1] - P[1] - dt * P[3],
                P[s1 + 2] - P[2] - dt * T * P[4], P[s1 + 3] - P[3] - dt * T * P[5],
                P[s1 + 7] - P[7] - dt * dt * alpha * (P[nx + 1] - P[nx]) - dt * dt * beta * (P[nx + 2] - P[nx + 3])]
    bx = [(-rx_max, rx_max), (-ry_max, ry_max), (-v_max, v_max), (-v_max, v_max)] + [(-1.0, 1.0)] * 4
    return _planar(N, 4, None, bx, (0.0, u_max), dyn,
                   lambda P, nx, nu: [P[nx + i] * (u_max - P[nx + i]) for i in range(nu)],
                   _state(x0, y0, vx0, vy0, theta0, theta_dot0, dt), _state(0.0, 0.0, 0.0, 0.0, 0.0, 0.0, dt),
                   Pf, fc_min, "flying")


PAPER_MODELS = {"cartpole": cartpole, "carback": carback, "landing": landing, "flying": flying}


# ----------------------------------------------------------------------------------------
# Rollouts (forward simulation of the printed discrete dynamics) in rescaled coordinates,
# for the invariant A(X(z)) = b and <C, X(z)> = sum f_k(z).
# ----------------------------------------------------------------------------------------
def planar_rollout(name: str, N: int, controls, **kw):
    """Landing / flying rollout from the model's initial state under `controls` (N x nu,
    physical units). Returns z in rescaled coordinates, in the global layout of `_planar`."""
    import numpy as np
    from math import sqrt
    pop = PAPER_MODELS[name](N=N, **kw)
    import inspect
    sig = inspect.signature(PAPER_MODELS[name])
    prm = {k: v.default for k, v in sig.parameters.items()}
    prm.update(kw)
    dt = prm["dt"]
    nu = 2 if name == "landing" else 4
    x = list(pop.meta["x_init"])
    zs = []
    for k in range(N):
        u = [float(c) for c in controls[k]]
        zs += x + u
        X, Y, VX, VY, RC, RS, FC, FS = x
        if name == "landing":
            T = u[0] + u[1]
            vx1 = VX - dt * T * RS / prm["m"]
            vy1 = VY + (dt * T * RC - dt * prm["m"] * prm["g"]) / prm["m"]
            fs1 = FS + prm["L"] * dt * dt * (u[1] - u[0]) / prm["Iz"]
        else:
            T = u[0] - u[1] + u[2] - u[3]
            vx1 = VX + dt * T * RC
            vy1 = VY + dt * T * RS
            fs1 = FS + dt * dt * prm["alpha"] * (u[1] - u[0]) + dt * dt * prm["beta"] * (u[2] - u[3])
        x = [X + dt * VX, Y + dt * VY, vx1, vy1, RC * FC - RS * FS, RS * FC + RC * FS, sqrt(1.0 - fs1 * fs1), fs1]
    zs += x
    # rescale with the model's boxes (same per variable type in every clique)
    bx = _planar_boxes(name, prm)
    box = bx[0] + [bx[1]] * nu
    out = []
    for i, v in enumerate(zs):
        lo, hi = box[i % (8 + nu)] if i < N * (8 + nu) else bx[0][i - N * (8 + nu)]
        out.append((v - (lo + hi) / 2) / ((hi - lo) / 2))
    return pop, np.asarray(out)


def _planar_boxes(name, prm):
    if name == "landing":
        bx = [(-prm["rx_max"], prm["rx_max"]), (prm["ry_min"], prm["ry_max"]), (-prm["v_max"], prm["v_max"]),
              (-prm["v_max"], prm["v_max"])] + [(-1.0, 1.0)] * 4
    else:
        bx = [(-prm["rx_max"], prm["rx_max"]), (-prm["ry_max"], prm["ry_max"]), (-prm["v_max"], prm["v_max"]),
              (-prm["v_max"], prm["v_max"])] + [(-1.0, 1.0)] * 4
    return bx, (0.0, prm["u_max"])


def carback_rollout(N: int, v, w, abc, x0: float = 2.0, y0: float = 4.0, theta0: float = 1.0,
                    dt: float = 0.25, ry_max: float = 8.0, v_max: float = 4.0, w_max: float = 0.5):
    """Car back-in rollout (eq:exp:cr:dis-dyn-constraints) under speeds v, turn rates w and
    unit separating-line vectors abc[k] = (A1, B1, C1, A2, B2, C2); rescaled z."""
    import numpy as np
    from math import sqrt
    rx_max = abs(x0) + 2.0
    x = [x0, y0, cos(theta0), sin(theta0)]
    sc_x = [rx_max, ry_max, 1.0, 1.0]
    sc_u = [v_max, w_max, 1.0, 1.0]
    z = []
    for k in range(N):
        fs = dt * w[k] - (dt * w[k]) ** 3 / 6.0
        fc = sqrt(1.0 - fs * fs)
        u = [v[k], w[k], fc, fs]
        z += [a / s for a, s in zip(x, sc_x)] + [a / s for a, s in zip(u, sc_u)] + list(abc[k])
        X, Y, RC, RS = x
        x = [X + dt * v[k] * RC, Y + dt * v[k] * RS, RC * fc - RS * fs, RS * fc + RC * fs]
    z += [a / s for a, s in zip(x, sc_x)]
    return np.asarray(z)


def paper_instance(name: str, N: int | None = None, seed: int = 0) -> ChainPop:
    """A seeded instance of one of the four models. The paper states no distribution of
    initial states for them; reading R-IS: seed 0 is the model's default
    start (cart-pole: the MPC start a = 0, theta = 0.1), seeds >= 1 draw
    uniformly from: cart-pole a0 in [-0.5, 0.5], theta0 in [0, pi], theta_dot0 in [-2, 2];
    car back-in x0 in [-8, 8], y0 in [2, 6] (above the gap), theta0 in [0, pi]; landing
    x0 in [-50, 50], y0 in [60, 110], velocities in [-5, 5], theta0 in [-0.3, 0.3];
    flying robot x0, y0 in [-8, 8], velocities in [-2, 2], theta0 in [-1, 1]."""
    import numpy as np
    fn = PAPER_MODELS[name]
    kw = {} if N is None else {"N": N}
    if seed == 0:
        return fn(**kw)
    r = np.random.default_rng(seed)
    U = lambda a, b: float(r.uniform(a, b))
    if name == "cartpole":
        kw.update(a0=U(-0.5, 0.5), theta0=U(0.0, pi), theta_dot0=U(-2.0, 2.0))
    elif name == "carback":
        kw.update(x0=U(-8.0, 8.0), y0=U(2.0, 6.0), theta0=U(0.0, pi))
    elif name == "landing":
        kw.update(x0=U(-50.0, 50.0), y0=U(60.0, 110.0), vx0=U(-5.0, 5.0), vy0=U(-5.0, 5.0), theta0=U(-0.3, 0.3))
    else:
        kw.update(x0=U(-8.0, 8.0), y0=U(-8.0, 8.0), vx0=U(-2.0, 2.0), vy0=U(-2.0, 2.0), theta0=U(-1.0, 1.0))
    return fn(**kw)
