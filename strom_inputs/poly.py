"""Monomials and polynomials in a clique's local variables.

Notation follows PAPER.md:100: a monomial z^alpha with alpha in N^d, its degree
sum(alpha); [z]_n the vector of monomials of degree <= n, of length
s(d, n) = C(n + d, d). Monomials are exponent tuples over the ordered clique
variables; [z]_n is in graded-lex order (degree major, then lexicographic in the
clique's variable order), which is the order of the paper's worked moment matrix
M_2 and of Example 2.
"""
from __future__ import annotations

import itertools
from math import comb
from typing import Dict, Iterable, List, Tuple

Mono = Tuple[int, ...]


def s_count(d: int, n: int) -> int:
    """s(d, n) = C(n + d, d)."""
    return comb(n + d, d)


def monomial_basis(nvars: int, deg: int) -> List[Mono]:
    """[z]_deg over `nvars` ordered variables, graded-lex."""
    out: List[Mono] = []
    for d in range(deg + 1):
        for combo in itertools.combinations_with_replacement(range(nvars), d):
            e = [0] * nvars
            for v in combo:
                e[v] += 1
            out.append(tuple(e))
    return out


def mono_add(a: Mono, b: Mono) -> Mono:
    return tuple(x + y for x, y in zip(a, b))


def mono_deg(a: Mono) -> int:
    return sum(a)


class Poly:
    """Sparse polynomial: {exponent tuple: coefficient}, no zero coefficients."""

    __slots__ = ("nvars", "terms")

    def __init__(self, nvars: int, terms: Dict[Mono, float] | None = None):
        self.nvars = nvars
        self.terms: Dict[Mono, float] = {}
        if terms:
            for m, c in terms.items():
                if c != 0.0:
                    self.terms[tuple(m)] = self.terms.get(tuple(m), 0.0) + float(c)
            self.terms = {m: c for m, c in self.terms.items() if c != 0.0}

    # --- constructors -------------------------------------------------
    @classmethod
    def const(cls, nvars: int, c: float) -> "Poly":
        return cls(nvars, {(0,) * nvars: c})

    @classmethod
    def var(cls, nvars: int, i: int, c: float = 1.0) -> "Poly":
        e = [0] * nvars
        e[i] = 1
        return cls(nvars, {tuple(e): c})

    # --- algebra --------------------------------------------------------
    def __add__(self, o) -> "Poly":
        if not isinstance(o, Poly):
            o = Poly.const(self.nvars, float(o))
        t = dict(self.terms)
        for m, c in o.terms.items():
            t[m] = t.get(m, 0.0) + c
        return Poly(self.nvars, t)

    __radd__ = __add__

    def __neg__(self) -> "Poly":
        return Poly(self.nvars, {m: -c for m, c in self.terms.items()})

    def __sub__(self, o) -> "Poly":
        if not isinstance(o, Poly):
            o = Poly.const(self.nvars, float(o))
        return self + (-o)

    def __rsub__(self, o) -> "Poly":
        return (-self) + o

    def __mul__(self, o) -> "Poly":
        if not isinstance(o, Poly):
            return Poly(self.nvars, {m: c * float(o) for m, c in self.terms.items()})
        t: Dict[Mono, float] = {}
        for m1, c1 in self.terms.items():
            for m2, c2 in o.terms.items():
                m = mono_add(m1, m2)
                t[m] = t.get(m, 0.0) + c1 * c2
        return Poly(self.nvars, t)

    __rmul__ = __mul__

    def __pow__(self, k: int) -> "Poly":
        out = Poly.const(self.nvars, 1.0)
        for _ in range(k):
            out = out * self
        return out

    # --- queries --------------------------------------------------------
    def degree(self) -> int:
        return max((mono_deg(m) for m in self.terms), default=0)

    def max_abs_coef(self) -> float:
        return max((abs(c) for c in self.terms.values()), default=0.0)

    def normalized(self) -> "Poly":
        """Divide by max |coef| (reading Q12(ii))."""
        s = self.max_abs_coef()
        return self * (1.0 / s) if s > 0 else self

    def eval(self, z: Iterable[float]) -> float:
        z = list(z)
        tot = 0.0
        for m, c in self.terms.items():
            v = c
            for zi, e in zip(z, m):
                if e:
                    v *= zi ** e
            tot += v
        return tot

    def support(self) -> set:
        s = set()
        for m in self.terms:
            s.update(i for i, e in enumerate(m) if e)
        return s

    def __repr__(self) -> str:  # pragma: no cover - debugging aid
        return f"Poly({self.terms})"
