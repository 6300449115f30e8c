"""Rank statistics of SURVEY §8(f) row f2 (Table 1; SPEC S:633-641 rank_stats).

Reporting only (host, float64): nothing here decides an ordering. The ranks come from the
library's exact fixed-point sums:
  centralized (p = 1):  D_i = T_i / (N 2^32), T_i = sum over all N sequences of q_ij
  globalized (f1):      D'_i = Dbar_i / 2^32, Dbar_i = floor(sum_s q(x_i, s) / m) over the m = p(p-1)
                        gathered samples
and R = ln(0.1 + D) (natural log: reading A4).
"""
from __future__ import annotations

import numpy as np

TWO32 = float(1 << 32)


def rank_R(D) -> np.ndarray:
    """R = ln(0.1 + D) (reading A4)."""
    return np.log(0.1 + np.asarray(D, dtype=np.float64))


def centralized_D(T, n: int) -> np.ndarray:
    """D_i = (1/N) sum_j r_ij from the fixed-point sum T_i (reading A5)."""
    return np.asarray(T, dtype=np.float64) / (n * TWO32)


def globalized_D(dbar) -> np.ndarray:
    """D'_i = Dbar_i / 2^32, the fixed-point mean similarity to the gathered samples."""
    return np.asarray(dbar, dtype=np.float64) / TWO32


def rank_stats(central, globalized) -> dict:
    """Table 1's fields: extrema and means of both rank vectors, and the
    population variance / standard deviation of (globalized - central) (SPEC S:633 decision D-Q1)."""
    a = np.asarray(central, dtype=np.float64)
    b = np.asarray(globalized, dtype=np.float64)
    if a.shape != b.shape or a.size == 0:
        raise ValueError("rank_stats needs two equally long, nonempty rank vectors")
    diff = b - a
    var = float(np.mean((diff - diff.mean()) ** 2))
    return {
        "(Maximum, Minimum) Central": (float(a.max()), float(a.min())),
        "Average Centralized": float(a.mean()),
        "(Maximum, Minimum) Globalized": (float(b.max()), float(b.min())),
        "Average Globalized": float(b.mean()),
        "Variance w.r.t. Centralized": var,
        "Standard Dev. w.r.t Centralized": float(np.sqrt(var)),
    }
