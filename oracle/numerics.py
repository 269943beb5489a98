"""ORACLE (test infrastructure only): float64 numerics of the mapped workloads.

The reference has no numeric model of the matmul workloads (SURVEY.md F9,
SPEC.md:8); per BASELINE.md section 4 the numeric oracle is numpy float64 on
the same (bf16-rounded) inputs.  Also serves as the `cpu_baseline` /
`--impl reference` leg of bench.py, on all host threads.
"""

from __future__ import annotations

import numpy as np


def sample_rows_cols(A: np.ndarray, Bt: np.ndarray) -> np.ndarray:
    """C = A @ Bt.T in float64 (A [r, K], Bt [c, K])."""
    return np.asarray(A, dtype=np.float64) @ np.asarray(Bt, dtype=np.float64).T


def jacobi5(grid: np.ndarray, sweeps: int) -> np.ndarray:
    """5-point Jacobi, fixed (Dirichlet) boundary, float64."""
    g = np.asarray(grid, dtype=np.float64).copy()
    for _ in range(sweeps):
        n = g.copy()
        n[1:-1, 1:-1] = 0.25 * (g[:-2, 1:-1] + g[2:, 1:-1] + g[1:-1, :-2] + g[1:-1, 2:])
        g = n
    return g
