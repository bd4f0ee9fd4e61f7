"""FP64 CPU oracle for Orthogonal Matching Pursuit — TEST INFRASTRUCTURE, NOT PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import or run anything under ``oracle/``.
The product path (``paper_2407_06434_b200``) never imports it and shares no
code with it.

What it computes: Algorithm 1 of the paper ("Orthogonal
Matching Pursuit"), one signal at a time, in plain FP64 numpy:

    initialization: x_0 = 0, r_0 = y
    for k = 1..S:
        n* = argmax_n |<r_{k-1}, a_n>| / ||a_n||
        S_k = S_{k-1} u {n*}
        x_k = argmin_x ||y - A_{S_k} x||
        r_k = y - A_{S_k} x_k
    or stop when ||y - A_{S_k} x_k|| <= eps

The least-squares step is solved FROM SCRATCH at every k by a Householder QR of
A_{S_k} (``numpy.linalg.qr``; PAPER.md:103 names QR as the alternative to
Cholesky), never incrementally, so it shares no structure with the
inverse-Cholesky update the CUDA path uses.

Readings of the paper where it is silent or ambiguous (DESIGN.md §2 lists them):
  R1  eps compares the residual NORM, inclusive (<=)
  R2  eps is tested before the first selection (r_0 = y)
  R3  S is a hard cap even when eps is given
  R4  argmax ties -> lowest atom index
  R5  selection divides by ||a_n|| on the raw A; the LS runs on the raw A, so
      x needs no rescale
  R6  stop with DEGENERATE (keeping the previous x) if n* is already selected,
      if the maximum correlation is 0, or if the new QR pivot collapses
  R15 the initial support S_0 is empty

Besides the result, every step records the diagnostics the parity protocol
needs: the top-two normalised correlations, the primary and
extended near-tie flags, the eps stop margin and the pivot ratio.

Pinned by tests/test_oracle_pins.py (P1-P11; P11 pins the per-step diagnostics and
first_flag() the parity protocol relies on); see DESIGN.md §4.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

# per-signal status codes (same numbering as the C ABI's ompSigStatus_t)
MAXITER = 0
EPS = 1
DEGENERATE = 2
NAN = 3

# near-tie / near-boundary thresholds (SURVEY §8(c) ambiguities 6, 8, 9; BASELINE.json north_star)
TIE_REL = 1e-5          # primary near-tie: t1 - t2 <= 1e-5 * t1
TIE_ABS_Y = 2e-6        # extended near-tie adds 2e-6 * ||y||
STOP_REL = 1e-5         # stop near-tie: | ||r_k|| - eps | <= 1e-5 * eps
QR_DEGENERATE = 1e-10   # min|diag R| <= 1e-10 * max|diag R|  -> DEGENERATE
NEAR_DEGENERATE = 1e-4  # pivot^2 < 1e-4 * ||a||^2               -> flagged step


@dataclass
class StepRecord:
    k: int                  # 1-based iteration index
    n_star: int             # selected atom (or the rejected one on a DEGENERATE step)
    t1: float               # largest  |<r_{k-1}, a_n>| / ||a_n||
    t2: float               # second largest over all other atoms
    primary_tie: bool       # t1 - t2 <= TIE_REL * t1
    extended_tie: bool      # t1 - t2 <= TIE_REL * t1 + TIE_ABS_Y * ||y||
    resid_norm: float       # ||r_k|| after the step (nan on a DEGENERATE step)
    stop_flag: bool         # | ||r_k|| - eps | <= STOP_REL * eps
    pivot_ratio: float      # R_kk^2 / ||a_{n*}||^2 of the QR of A_{S_k}
    near_degenerate: bool   # pivot_ratio < NEAR_DEGENERATE


@dataclass
class OracleResult:
    support: np.ndarray               # (n_iter,) int64, selection order
    x: np.ndarray                     # (n_iter,) float64, coefficient of support[j]
    resid_norm: float
    n_iter: int
    status: int
    y_norm: float
    eps: Optional[float]
    init_stop_flag: bool = False      # | ||y|| - eps | <= STOP_REL * eps at k = 0
    steps: List[StepRecord] = field(default_factory=list)

    def dense(self, N: int) -> np.ndarray:
        out = np.zeros(N)
        out[self.support] = self.x
        return out

    def first_flag(self, extended: bool = False) -> Optional[int]:
        """0-based index of the first step whose selection or stop decision is flagged."""
        if self.init_stop_flag:
            return 0
        for i, s in enumerate(self.steps):
            tie = s.extended_tie if extended else s.primary_tie
            if tie or s.stop_flag or s.near_degenerate:
                return i
        return None


def atom_norms(A64: np.ndarray) -> np.ndarray:
    """||a_n|| for every column (PAPER.md:46 denominator).  Rejects zero or non-finite columns."""
    if not np.all(np.isfinite(A64)):
        bad = int(np.argwhere(~np.isfinite(A64))[0][1])
        raise ValueError(f"non-finite entry in dictionary column {bad}")
    nrm = np.sqrt(np.sum(A64 * A64, axis=0))
    if np.any(nrm == 0):
        raise ValueError(f"zero-norm dictionary column {int(np.argmin(nrm))}")
    return nrm


def _no_eps(eps) -> bool:
    return eps is None or (isinstance(eps, float) and math.isnan(eps)) or eps < 0


def omp(A, y, S: int, eps: Optional[float] = None, norms: Optional[np.ndarray] = None) -> OracleResult:
    """Algorithm 1 on one signal, FP64, LS re-solved by QR at every step."""
    A64 = np.asarray(A, dtype=np.float64)
    y64 = np.asarray(y, dtype=np.float64)
    M, N = A64.shape
    if not (1 <= S <= min(M, N)):
        raise ValueError("need 1 <= S <= min(M, N)")
    nrm = atom_norms(A64) if norms is None else norms
    use_eps = not _no_eps(eps)

    if not np.all(np.isfinite(y64)):
        return OracleResult(np.zeros(0, np.int64), np.zeros(0), float("nan"), 0, NAN,
                            float("nan"), eps if use_eps else None)

    y_norm = float(np.linalg.norm(y64))
    res = OracleResult(np.zeros(0, np.int64), np.zeros(0), y_norm, 0, MAXITER, y_norm,
                       eps if use_eps else None)
    # initialization: x_0 = 0, r_0 = y; reading R2: test eps on r_0
    if use_eps:
        res.init_stop_flag = abs(y_norm - eps) <= STOP_REL * eps
        if y_norm <= eps:
            res.status = EPS
            return res

    support: List[int] = []
    x = np.zeros(0)
    r = y64.copy()
    for k in range(1, S + 1):
        # n* = argmax_n |<r_{k-1}, a_n>| / ||a_n||; np.argmax -> lowest index on ties
        t = np.abs(A64.T @ r) / nrm
        n_star = int(np.argmax(t))
        t1 = float(t[n_star])
        t2 = float(np.max(np.delete(t, n_star))) if N > 1 else 0.0
        gap = t1 - t2
        primary = gap <= TIE_REL * t1
        extended = gap <= TIE_REL * t1 + TIE_ABS_Y * y_norm
        # reading R6: re-selection or an exhausted residual ends the signal
        if n_star in support or t1 == 0.0:
            res.steps.append(StepRecord(k, n_star, t1, t2, primary, extended, float("nan"),
                                        False, 0.0, True))
            res.status = DEGENERATE
            break
        # S_k = S_{k-1} u {n*}
        cand = support + [n_star]
        A_S = A64[:, cand]
        # x_k = argmin ||y - A_{S_k} x||, by Householder QR from scratch
        Q, R = np.linalg.qr(A_S, mode="reduced")
        diag = np.abs(np.diag(R))
        pivot_ratio = float(diag[-1] ** 2 / (nrm[n_star] ** 2))
        if diag.min() <= QR_DEGENERATE * diag.max():
            res.steps.append(StepRecord(k, n_star, t1, t2, primary, extended, float("nan"),
                                        False, pivot_ratio, True))
            res.status = DEGENERATE
            break
        x_new = np.linalg.solve(np.triu(R), Q.T @ y64)
        # r_k = y - A_{S_k} x_k
        r = y64 - A_S @ x_new
        rn = float(np.linalg.norm(r))
        support, x = cand, x_new
        stop_flag = use_eps and abs(rn - eps) <= STOP_REL * eps
        res.steps.append(StepRecord(k, n_star, t1, t2, primary, extended, rn, stop_flag,
                                    pivot_ratio, pivot_ratio < NEAR_DEGENERATE))
        res.resid_norm = rn
        # or stop when ||y - A_{S_k} x_k|| <= eps
        if use_eps and rn <= eps:
            res.status = EPS
            break
    res.support = np.asarray(support, dtype=np.int64)
    res.x = np.asarray(x, dtype=np.float64)
    res.n_iter = len(support)
    return res


# ----------------------------------------------------------------------------------------
# batch driver: one worker process per host core, one BLAS thread each
# ----------------------------------------------------------------------------------------

_W = {}


def _worker_init(A, S, eps):
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        pass
    A64 = np.asarray(A, dtype=np.float64)
    _W["A"], _W["S"], _W["eps"], _W["nrm"] = A64, S, eps, atom_norms(A64)


def _worker_run(Yc):
    return [omp(_W["A"], y, _W["S"], _W["eps"], _W["nrm"]) for y in Yc]


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def omp_batch(A, Y, S: int, eps: Optional[float] = None, workers: Optional[int] = None,
              chunk: Optional[int] = None) -> List[OracleResult]:
    """Run :func:`omp` on every row of Y (shape (B, M)); rows are independent signals."""
    Y = np.asarray(Y)
    B = Y.shape[0]
    workers = host_cores() if workers is None else max(1, int(workers))
    workers = min(workers, B) if B > 0 else 1
    if workers <= 1 or B <= 2:
        A64 = np.asarray(A, dtype=np.float64)
        nrm = atom_norms(A64)
        return [omp(A64, y, S, eps, nrm) for y in Y]
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    if chunk is None:
        chunk = max(1, -(-B // (workers * 4)))
    parts = [Y[i:i + chunk] for i in range(0, B, chunk)]
    ctx = mp.get_context("fork")
    # the workers get A exactly as given (promoted to FP64 by _worker_init, like the serial path)
    with ProcessPoolExecutor(max_workers=workers, mp_context=ctx, initializer=_worker_init,
                             initargs=(np.asarray(A), S, eps)) as ex:
        out: List[OracleResult] = []
        for part in ex.map(_worker_run, parts):
            out.extend(part)
    return out


def least_squares_residual(A, y, support: Sequence[int]) -> float:
    """||y - A_T x_T|| for the LS solution on support T (helper for the brute-force pins)."""
    A64 = np.asarray(A, dtype=np.float64)
    y64 = np.asarray(y, dtype=np.float64)
    if len(support) == 0:
        return float(np.linalg.norm(y64))
    A_T = A64[:, list(support)]
    xt, *_ = np.linalg.lstsq(A_T, y64, rcond=None)
    return float(np.linalg.norm(y64 - A_T @ xt))
