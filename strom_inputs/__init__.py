"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package is the *input side* of the build (SURVEY.md §1 layer L0/L1): the
polynomial trajectory-optimisation models of the paper and
STROM's primal sparse moment relaxation compiler, which turns
a chain-sparse POP into the standard multi-block SDP

    min <C, X>  s.t.  A(X) = b,  X in Omega_+          

It holds NONE of the sGS-ADMM arithmetic (no A/A* products, no projection, no
linear solve, no residuals): both `oracle/` and the CUDA path consume the SDP
bytes produced here, so both see identical inputs (SURVEY.md §8(b) "What the
library does not do").
"""
from .poly import Poly, monomial_basis, s_count
from .relax import ChainPop, BlockSdp, compile_relaxation, lift_rank1, svec_index
from . import models

__all__ = [
    "Poly", "monomial_basis", "s_count", "ChainPop", "BlockSdp",
    "compile_relaxation", "lift_rank1", "svec_index", "models",
]
