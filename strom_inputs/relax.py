"""STROM's primal sparse moment relaxation compiler.

Turns a chain-sparse POP (Definition 1) into the standard
multi-block SDP  min <C,X>  s.t.  A(X) = b,  X in Omega_+  
whose blocks are the moment matrices M_k (order s(|I_k|, kappa)) and the
localizing matrices L_{k,i} (order s(|I_k|, kappa - d_g)) of the relaxation
(PAPER.md:254-258).

Readings (listed again in DESIGN.md):
  * svec (Q4): SDPT3 convention -- upper triangle column-wise, off-diagonal
    entries scaled by sqrt(2), so <A,B> = svec(A).svec(B).
  * canonical occurrence (Q5): the first occurrence of a monomial in svec
    order; every other occurrence is equated to it (A_mom), and
    localizing / equality / consensus rows address canonical occurrences only.
  * normalisation (Q6): once, M_1(1,1) = 1, with the constant monomial included
    in the consensus rows.
  * row order: clique-major, family-minor (norm, mom, ineq, eq, sen), blocks
    ordered clique-major (M_k then L_{k,i}) -- "we sort matrix variables and
    linear constraints by clique indices".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil, sqrt
from typing import Dict, List, Sequence

import numpy as np

from .poly import Mono, Poly, monomial_basis, mono_add

FAMILY_NORM, FAMILY_MOM, FAMILY_INEQ, FAMILY_EQ, FAMILY_SEN = 0, 1, 2, 3, 4
KIND_MOMENT, KIND_LOCALIZING = 0, 1
_ISQ2 = 1.0 / sqrt(2.0)


def svec_index(r: int, c: int) -> int:
    """Position of upper-triangular entry (r, c), r <= c, column-wise (Q4)."""
    if r > c:
        r, c = c, r
    return c * (c + 1) // 2 + r


def svec_len(n: int) -> int:
    return n * (n + 1) // 2


@dataclass
class ChainPop:
    """Chain-sparse POP (eq:strom:popsdp:chain-sparse-pop).

    cliques[k] is the ordered list of global variable indices I_k; f[k], g[k][i],
    h[k][j] are Polys in the clique-local variables of I_k. R[k] bounds
    ||z(I_k)||_inf (Theorem 1/2 assumption).
    """
    d: int
    cliques: List[List[int]]
    f: List[Poly]
    g: List[List[Poly]]
    h: List[List[Poly]]
    R: List[float]
    name: str = "pop"
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return len(self.cliques)

    def objective(self, z: Sequence[float]) -> float:
        z = np.asarray(z, dtype=np.float64)
        return float(sum(fk.eval(z[I]) for fk, I in zip(self.f, self.cliques)))

    def validate_chain(self) -> List[str]:
        """Violations of eq:strom:popsdp:index-chainrule."""
        errs = []
        cover = set()
        for k, I in enumerate(self.cliques):
            if k >= 1:
                prev = set().union(*[set(J) for J in self.cliques[:k]])
                if prev & set(I) != set(self.cliques[k - 1]) & set(I):
                    errs.append(f"chain rule broken at clique {k}")
            cover |= set(I)
            for p in [self.f[k], *self.g[k], *self.h[k]]:
                if p.nvars != len(I):
                    errs.append(f"poly arity mismatch in clique {k}")
        if cover != set(range(self.d)):
            errs.append("cliques do not cover all variables")
        return errs


@dataclass
class BlockSdp:
    """Standard multi-block SDP data in svec coordinates.

    A is stored as CSR over rows (indptr int64, indices int32 global svec column,
    data float64). Blocks are clique-major; block_offset gives each block's svec
    start.
    """
    block_n: np.ndarray        # int32 [nblocks] matrix order n_beta
    block_stage: np.ndarray    # int32 [nblocks] clique k (0-based)
    block_kind: np.ndarray     # int8  [nblocks] 0 moment, 1 localizing
    block_offset: np.ndarray   # int64 [nblocks+1]
    A_indptr: np.ndarray       # int64 [m+1]
    A_indices: np.ndarray      # int32 [nnz]
    A_data: np.ndarray         # float64 [nnz]
    b: np.ndarray              # float64 [m]
    C: np.ndarray              # float64 [n]
    row_family: np.ndarray     # int8  [m]
    row_stage: np.ndarray      # int32 [m]  (consensus rows: left clique)
    R_beta: np.ndarray         # float64 [nblocks] trace bounds (Theorem 2)
    kappa: int = 2
    name: str = "sdp"
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.block_offset[-1])

    @property
    def m(self) -> int:
        return int(self.b.shape[0])

    @property
    def nblocks(self) -> int:
        return int(self.block_n.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.A_indices.shape[0])

    def summary(self) -> dict:
        mom = self.block_n[self.block_kind == KIND_MOMENT]
        loc = self.block_n[self.block_kind == KIND_LOCALIZING]
        return {
            "name": self.name, "n": self.n, "m": self.m, "nnz": self.nnz,
            "moment_blocks": int(mom.size), "moment_order": sorted(set(mom.tolist())),
            "localizing_blocks": int(loc.size), "localizing_order": sorted(set(loc.tolist())),
        }

    def save(self, path: str) -> None:
        np.savez(path, **{k: getattr(self, k) for k in _ARRAYS},
                 kappa=self.kappa, name=self.name)

    @classmethod
    def load(cls, path: str) -> "BlockSdp":
        z = np.load(path, allow_pickle=False)
        return cls(**{k: z[k] for k in _ARRAYS}, kappa=int(z["kappa"]), name=str(z["name"]))


_ARRAYS = ["block_n", "block_stage", "block_kind", "block_offset", "A_indptr",
           "A_indices", "A_data", "b", "C", "row_family", "row_stage", "R_beta"]


class _CliqueTable:
    """Per-clique monomial bookkeeping: basis, svec entries, canonical map."""

    def __init__(self, nvars: int, kappa: int):
        self.nvars = nvars
        self.basis = monomial_basis(nvars, kappa)
        nM = len(self.basis)
        self.nM = nM
        self.canon: Dict[Mono, int] = {}
        self.occ: Dict[Mono, List[int]] = {}
        self.entry_coef = np.empty(svec_len(nM))
        for c in range(nM):
            for r in range(c + 1):
                s = svec_index(r, c)
                mono = mono_add(self.basis[r], self.basis[c])
                if mono not in self.canon:
                    self.canon[mono] = s
                    self.occ[mono] = [s]
                else:
                    self.occ[mono].append(s)
                self.entry_coef[s] = 1.0 if r == c else _ISQ2


def _entry_coef(r: int, c: int) -> float:
    return 1.0 if r == c else _ISQ2


class _LazyCanon:
    """meta["canon"][k] built on first use (the C++ generator does not return the maps)."""

    def __init__(self, pop, kappa):
        self.pop, self.kappa, self.cache = pop, kappa, {}

    def __getitem__(self, k):
        if k not in self.cache:
            self.cache[k] = _CliqueTable(len(self.pop.cliques[k]), self.kappa).canon
        return self.cache[k]

    def __len__(self):
        return self.pop.N


def compile_relaxation(pop: ChainPop, kappa: int = 2, name: str | None = None,
                       normalize: bool = True, engine: str | None = None) -> BlockSdp:
    """The relaxation as a BlockSdp. engine "cpp" (default when strom_inputs/libstrom_gen.so
    loads: the C++ generator of NEXT-3, per clique in parallel) or "python" (the reference
    implementation below; STROM_GEN=python forces it). Both produce identical bytes."""
    import os
    engine = engine or os.environ.get("STROM_GEN", "cpp")
    if engine == "cpp":
        from . import fastgen
        if fastgen.available():
            return _compile_cpp(pop, kappa, name, normalize)
    return compile_relaxation_py(pop, kappa, name, normalize)


def _compile_cpp(pop: ChainPop, kappa: int, name, normalize: bool) -> BlockSdp:
    from . import fastgen
    N = pop.N
    gs = [[(gi.normalized() if normalize else gi) for gi in pop.g[k]] for k in range(N)]
    hs = [[(hj.normalized() if normalize else hj) for hj in pop.h[k]] for k in range(N)]
    arr = fastgen.compile_arrays(pop, kappa, gs, hs)
    basis = [monomial_basis(len(I), kappa) for I in pop.cliques]
    mom_block, loc_blocks, loc_bases = [], [], []
    bi = 0
    for k in range(N):
        mom_block.append(bi); bi += 1
        lb, lbas = [], []
        for gi in gs[k]:
            lb.append(bi); bi += 1
            lbas.append(monomial_basis(len(pop.cliques[k]), kappa - ceil(gi.degree() / 2)))
        loc_blocks.append(lb); loc_bases.append(lbas)
    R_beta = _trace_bounds(pop, kappa, normalize, gs, [len(B) for B in basis], mom_block, loc_blocks, loc_bases,
                           len(arr["block_n"]))
    sdp = BlockSdp(R_beta=R_beta, kappa=kappa, name=name or pop.name, **arr)
    sdp.meta = {"mom_block": mom_block, "loc_blocks": loc_blocks, "basis": basis, "loc_bases": loc_bases,
                "canon": _LazyCanon(pop, kappa), "g_normalized": gs, "pop": pop}
    return sdp


def _trace_bounds(pop, kappa, normalize, gs, nM, mom_block, loc_blocks, loc_bases, nblocks):
    """R_beta (Theorem 2; reading Q17)."""
    R_beta = np.empty(nblocks)
    for k in range(pop.N):
        Rk = max(1.0, float(pop.R[k]))
        R_beta[mom_block[k]] = nM[k] * Rk ** (2 * kappa)
        gmax = pop.meta.get("gmax")
        for i, gi in enumerate(gs[k]):
            dg = ceil(gi.degree() / 2)
            if gmax is not None:
                gm = gmax[k][i] / (pop.g[k][i].max_abs_coef() if normalize else 1.0)
            else:  # sum |coef| * Rk^deg bounds max g over the box
                gm = sum(abs(c) * Rk ** sum(a) for a, c in gi.terms.items())
            R_beta[loc_blocks[k][i]] = max(gm, 0.0) * len(loc_bases[k][i]) * Rk ** (2 * (kappa - dg))
    return R_beta


def compile_relaxation_py(pop: ChainPop, kappa: int = 2, name: str | None = None,
                          normalize: bool = True) -> BlockSdp:
    """kappa-th order sparse moment relaxation as a standard SDP.

    Row families per clique k:
      norm  M_1(1,1) = 1                                  (eq. ...-normalize)
      mom   occurrence_j - canonical = 0                  (A_mom)
      ineq  L(r,c) - sum_a g_a M(canon(a+B_r+B_c)) = 0     (A_ineq)
      eq    sum_a h_a M(canon(a+mu)) = 0, mu in [z]_{2k-deg h} (A_eq)
      sen   canon_k(mono) - canon_{k+1}(mono) = 0          (A_sen)
    If `normalize`, every g and h is divided by its max |coef| first (Q12(ii)).
    """
    N = pop.N
    tables = [_CliqueTable(len(I), kappa) for I in pop.cliques]
    gs = [[(gi.normalized() if normalize else gi) for gi in pop.g[k]] for k in range(N)]
    hs = [[(hj.normalized() if normalize else hj) for hj in pop.h[k]] for k in range(N)]

    # ---- blocks -----------------------------------------------------------
    block_n, block_stage, block_kind, R_beta = [], [], [], []
    mom_block, loc_blocks = [], []
    loc_bases = []
    for k in range(N):
        mom_block.append(len(block_n))
        block_n.append(tables[k].nM); block_stage.append(k); block_kind.append(KIND_MOMENT)
        R_beta.append(np.nan)
        lb, lbas = [], []
        for gi in gs[k]:
            dg = ceil(gi.degree() / 2)
            if dg > kappa:
                raise ValueError("unsupported-degree: 2*ceil(deg g/2) > 2*kappa")
            B1 = monomial_basis(len(pop.cliques[k]), kappa - dg)
            lb.append(len(block_n)); lbas.append(B1)
            block_n.append(len(B1)); block_stage.append(k); block_kind.append(KIND_LOCALIZING)
            R_beta.append(np.nan)
        loc_blocks.append(lb); loc_bases.append(lbas)
    block_n = np.asarray(block_n, dtype=np.int32)
    block_offset = np.zeros(len(block_n) + 1, dtype=np.int64)
    block_offset[1:] = np.cumsum(block_n.astype(np.int64) * (block_n + 1) // 2)
    n = int(block_offset[-1])

    # ---- rows -------------------------------------------------------------
    rows_cols: List[np.ndarray] = []
    rows_vals: List[np.ndarray] = []
    fam: List[int] = []
    stage: List[int] = []
    b_list: List[float] = []

    def emit(entries: Dict[int, float], family: int, k: int, rhs: float = 0.0):
        ent = {c: v for c, v in entries.items() if v != 0.0}
        if not ent:
            return
        cols = np.fromiter(sorted(ent), dtype=np.int64)
        rows_cols.append(cols)
        rows_vals.append(np.asarray([ent[c] for c in cols.tolist()], dtype=np.float64))
        fam.append(family); stage.append(k); b_list.append(rhs)

    for k in range(N):
        T = tables[k]
        offM = int(block_offset[mom_block[k]])
        ec = T.entry_coef
        # norm
        if k == 0:
            emit({offM + 0: 1.0}, FAMILY_NORM, k, 1.0)
        # mom: monomials in order of canonical svec position
        for mono, lst in sorted(T.occ.items(), key=lambda kv: kv[1][0]):
            s0 = lst[0]
            for sj in lst[1:]:
                emit({offM + sj: ec[sj], offM + s0: -ec[s0]}, FAMILY_MOM, k)
        # ineq
        for i, gi in enumerate(gs[k]):
            offL = int(block_offset[loc_blocks[k][i]])
            B1 = loc_bases[k][i]
            nL = len(B1)
            for c in range(nL):
                for r in range(c + 1):
                    ent: Dict[int, float] = {offL + svec_index(r, c): _entry_coef(r, c)}
                    base = mono_add(B1[r], B1[c])
                    for a, ga in gi.terms.items():
                        s = T.canon[mono_add(a, base)]
                        ent[offM + s] = ent.get(offM + s, 0.0) - ga * ec[s]
                    emit(ent, FAMILY_INEQ, k)
        # eq
        for hj in hs[k]:
            dh = hj.degree()
            if dh > 2 * kappa:
                raise ValueError("order-too-low: deg h > 2 kappa")
            for mu in monomial_basis(T.nvars, 2 * kappa - dh):
                ent = {}
                for a, ha in hj.terms.items():
                    s = T.canon[mono_add(a, mu)]
                    ent[offM + s] = ent.get(offM + s, 0.0) + ha * ec[s]
                emit(ent, FAMILY_EQ, k)
        # sen with clique k+1
        if k + 1 < N:
            I0, I1 = pop.cliques[k], pop.cliques[k + 1]
            shared = [v for v in I0 if v in set(I1)]
            T1 = tables[k + 1]
            offM1 = int(block_offset[mom_block[k + 1]])
            pos0 = [I0.index(v) for v in shared]
            pos1 = [I1.index(v) for v in shared]
            for ms in monomial_basis(len(shared), 2 * kappa):
                e0 = [0] * len(I0); e1 = [0] * len(I1)
                for j, p in enumerate(ms):
                    e0[pos0[j]] += p; e1[pos1[j]] += p
                s0 = T.canon[tuple(e0)]; s1 = T1.canon[tuple(e1)]
                emit({offM + s0: ec[s0], offM1 + s1: -T1.entry_coef[s1]}, FAMILY_SEN, k)

    m = len(b_list)
    lens = np.fromiter((len(c) for c in rows_cols), dtype=np.int64, count=m)
    indptr = np.zeros(m + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(lens)
    indices = np.concatenate(rows_cols).astype(np.int32)
    data = np.concatenate(rows_vals)

    # ---- objective (canonical occurrences, reading Q11) ----------------------
    C = np.zeros(n)
    for k in range(N):
        T = tables[k]
        offM = int(block_offset[mom_block[k]])
        for a, fa in pop.f[k].terms.items():
            s = T.canon[a]
            C[offM + s] += fa * T.entry_coef[s]

    # ---- trace bounds R_beta (Theorem 2; reading Q17) ---
    R_beta = _trace_bounds(pop, kappa, normalize, gs, [T.nM for T in tables], mom_block, loc_blocks,
                           loc_bases, len(block_n))

    sdp = BlockSdp(
        block_n=block_n,
        block_stage=np.asarray(block_stage, dtype=np.int32),
        block_kind=np.asarray(block_kind, dtype=np.int8),
        block_offset=block_offset,
        A_indptr=indptr, A_indices=indices, A_data=data,
        b=np.asarray(b_list, dtype=np.float64), C=C,
        row_family=np.asarray(fam, dtype=np.int8),
        row_stage=np.asarray(stage, dtype=np.int32),
        R_beta=R_beta, kappa=kappa, name=name or pop.name,
    )
    sdp.meta = {
        "mom_block": mom_block, "loc_blocks": loc_blocks,
        "basis": [T.basis for T in tables], "loc_bases": loc_bases,
        "canon": [T.canon for T in tables], "g_normalized": gs, "pop": pop,
    }
    return sdp


def lift_rank1(sdp: BlockSdp, z: Sequence[float]) -> np.ndarray:
    """X(z): M_k(z) = [z]_k[z]_k^T, L_{k,i}(z) = g [z]_{k-d}[z]_{k-d}^T, in svec
    (eq:strom:sgsadmm:rank1-lifting)."""
    pop: ChainPop = sdp.meta["pop"]
    z = np.asarray(z, dtype=np.float64)
    X = np.zeros(sdp.n)
    for k, I in enumerate(pop.cliques):
        zk = z[I]
        blocks = [(sdp.meta["mom_block"][k], sdp.meta["basis"][k], 1.0)]
        for i, gi in enumerate(sdp.meta["g_normalized"][k]):
            blocks.append((sdp.meta["loc_blocks"][k][i], sdp.meta["loc_bases"][k][i], gi.eval(zk)))
        for bi, B, w in blocks:
            v = np.array([np.prod(zk ** np.asarray(e)) for e in B])
            Mz = w * np.outer(v, v)
            nb = len(B)
            off = int(sdp.block_offset[bi])
            for c in range(nb):
                for r in range(c + 1):
                    X[off + svec_index(r, c)] = Mz[r, c] * (1.0 if r == c else sqrt(2.0))
    return X
