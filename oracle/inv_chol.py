"""Inverse-Cholesky least-squares update of the paper's "algorithm v0" — TEST INFRASTRUCTURE.

Written out step by step from PAPER.md:133-177 (Section 2.2), FP64, dense
matrices, no packing and no fusion:

    F_1 := 1 / ||a_{n*}||                                            (Eq. 7)
    F_k := [[F_{k-1}, -gamma F_{k-1} z], [0, gamma]]                  (Eq. 8)
    z    = F_{k-1}^T A_{k-1}^T a_{n*}
    gamma = 1 / sqrt(||a_{n*}||^2 - ||z||^2)
    F_k V_k^T = I  =>  F_k = V_k^{-T}
    x_hat = F_k F_k^T A_k^T y                                         (Eq. 11)

and the Cholesky-update route it is equivalent to (Eqs. 4-6):

    V_1 := ||a_{n*}||,  V_k := [[V_{k-1}, 0], [z^T, sqrt(||a||^2 - ||z||^2)]],  V_{k-1} z = A_{k-1}^T a_{n*}

This module is a second, independent statement of what the CUDA path's
factor-append kernel (K3) computes.  Its identities are pinned against
``numpy.linalg.cholesky`` / ``numpy.linalg.qr`` (tests/test_oracle_pins.py, P5/P9).
It is used only by tests/.
"""

from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np


def inv_chol_append(F_prev: Optional[np.ndarray], w: np.ndarray, d: float) -> Tuple[np.ndarray, np.ndarray, float]:
    """One step of Eqs. (7)-(8).

    F_prev: k-1 x k-1 upper-triangular F_{k-1} (None for k = 1)
    w:      A_{k-1}^T a_{n*}  (length k-1; the Gram entries [A^T A]_{n*, S})
    d:      ||a_{n*}||^2
    returns (F_k, z, gamma)
    """
    if F_prev is None or F_prev.size == 0:
        gamma = 1.0 / np.sqrt(d)                      # Eq. 7: F_1 = 1/||a_{n*}||
        return np.array([[gamma]]), np.zeros(0), float(gamma)
    z = F_prev.T @ w                                   # z = F_{k-1}^T A_{k-1}^T a_{n*}
    delta = d - z @ z
    if delta <= 0:
        raise np.linalg.LinAlgError("rank deficiency: ||a||^2 - ||z||^2 <= 0")
    gamma = 1.0 / np.sqrt(delta)                       # gamma = 1/sqrt(||a||^2 - ||z||^2)
    k = F_prev.shape[0] + 1
    F = np.zeros((k, k))
    F[:k - 1, :k - 1] = F_prev
    F[:k - 1, k - 1] = -gamma * (F_prev @ z)           # -gamma F_{k-1} z
    F[k - 1, k - 1] = gamma
    return F, z, float(gamma)


def chol_append(V_prev: Optional[np.ndarray], w: np.ndarray, d: float) -> np.ndarray:
    """Eqs. (4)-(5): lower-triangular V_k from V_{k-1} (forward substitution for z)."""
    if V_prev is None or V_prev.size == 0:
        return np.array([[np.sqrt(d)]])
    k1 = V_prev.shape[0]
    z = np.zeros(k1)
    for i in range(k1):                                 # solve V_{k-1} z = A_{k-1}^T a_{n*}
        z[i] = (w[i] - V_prev[i, :i] @ z[:i]) / V_prev[i, i]
    V = np.zeros((k1 + 1, k1 + 1))
    V[:k1, :k1] = V_prev
    V[k1, :k1] = z
    V[k1, k1] = np.sqrt(d - z @ z)
    return V


def ls_by_inverse_cholesky(A, y, support) -> Tuple[np.ndarray, List[np.ndarray], List[float]]:
    """x_hat on a fixed support sequence via Eqs. (7), (8), (11); also returns F_k and gamma_k per step."""
    A64 = np.asarray(A, dtype=np.float64)
    y64 = np.asarray(y, dtype=np.float64)
    F = None
    Fs, gammas = [], []
    for k in range(1, len(support) + 1):
        a = A64[:, support[k - 1]]
        A_prev = A64[:, list(support[:k - 1])]
        F, _, g = inv_chol_append(F, A_prev.T @ a, float(a @ a))
        Fs.append(F)
        gammas.append(g)
    A_k = A64[:, list(support)]
    x = F @ (F.T @ (A_k.T @ y64))                      # Eq. 11: x = F_k F_k^T A_k^T y
    return x, Fs, gammas
