"""ORACLE -- test infrastructure, NOT part of the product.

A plain, slow, obviously-correct CPU fp64 implementation of what the sGS-ADMM
hot path computes (Algorithm 1), written from the paper and
sharing no code with the CUDA path (`paper_2406_05846_b200/`). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import it.

Pins: see tests/test_oracle_*.py. Every function states the passage it follows.
"""
from .admm import (Oracle, OracleConfig, svec_to_mat, mat_to_svec, project_psd_block,
                   kkt_residuals, sigma_update)
from .certificate import lower_bound, extract_pendulum, suboptimality_gap

__all__ = ["Oracle", "OracleConfig", "svec_to_mat", "mat_to_svec", "project_psd_block",
           "kkt_residuals", "sigma_update", "lower_bound", "extract_pendulum",
           "suboptimality_gap"]
