"""Exhaustive best-support search — TEST INFRASTRUCTURE, NOT PRODUCT.

PAPER.md:66-71: OMP greedily approximates
    argmin_x ||A x - y||  s.t. |supp x| <= S,
whose exact solution needs all N!/(S!(N-S)!) supports; "it does not necessarily
converge to the global optimum".  This module enumerates every size-S support
of a tiny dictionary (pin P4): it ranks all supports by the normal-equation
objective ||y||^2 - b_T^T (A_T^T A_T)^{-1} b_T (b_T = A_T^T y), then recomputes
the best few by ``numpy.linalg.lstsq`` because that shortcut loses about
sqrt(machine eps) to cancellation.

Only tests/ may import this.
"""

from __future__ import annotations

import itertools
from math import comb
from typing import Tuple

import numpy as np


def all_supports(N: int, S: int) -> np.ndarray:
    if comb(N, S) > 2_000_000:
        raise ValueError(f"C({N},{S}) = {comb(N, S)} supports exceeds the exhaustive-search budget")
    return np.fromiter(itertools.chain.from_iterable(itertools.combinations(range(N), S)),
                       dtype=np.int64).reshape(-1, S)


def exhaustive_best_support(A, y, S: int, recheck: int = 32) -> Tuple[np.ndarray, float]:
    """Return (support, ||y - A_T x_T||) of the globally optimal size-S support (lexicographic ties)."""
    A64 = np.asarray(A, dtype=np.float64)
    y64 = np.asarray(y, dtype=np.float64)
    N = A64.shape[1]
    T = all_supports(N, S)
    G = A64.T @ A64
    b = A64.T @ y64
    GT = G[T[:, :, None], T[:, None, :]]
    bT = b[T]
    sol = np.linalg.solve(GT, bT[..., None])[..., 0]
    obj = float(y64 @ y64) - np.sum(bT * sol, axis=1)
    order = np.argsort(obj, kind="stable")[:recheck]
    best, best_r = None, np.inf
    for i in order:
        A_T = A64[:, T[i]]
        xt, *_ = np.linalg.lstsq(A_T, y64, rcond=None)
        rr = float(np.linalg.norm(y64 - A_T @ xt))
        if rr < best_r:
            best, best_r = T[i], rr
    return np.asarray(best), best_r
