"""Parity protocol: CUDA results vs the FP64 oracle, per signal (SURVEY §8(c) "Parity protocol").

Tolerances (BASELINE.json north_star; readings R10/R11):
  * supports: identical selection sequence, n_iter and status, unless the oracle
    flags the step (primary near-tie t1-t2 <= 1e-5 t1, eps stop near-boundary,
    near-degenerate pivot);
  * coefficients: ||x_gpu - x_ora||_2 / ||x_ora||_2 <= 1e-4 over dense N-vectors
    aligned by atom index (x_ora = 0 requires x_gpu = 0 exactly);
  * residual norm: | r_gpu - r_ora | <= 1e-4 r_ora + 1e-5 ||y||.

Outcome per signal:
  "exact"          unflagged, sequences identical, values within tolerance
  "flagged_ok"     flagged, decisions before the flag identical, same final support
                   set, values within tolerance
  "tie_divergent"  flagged, supports diverge after the flag (reported, not failed)
  "explained"      diverges at a step only the EXTENDED near-tie rule flags
  "bug"            anything else (must be 0)
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

COEF_RTOL = 1e-4
RES_RTOL = 1e-4
RES_ATOL_Y = 1e-5
NAN_STATUS = 3


@dataclass
class GpuSignal:
    support: np.ndarray   # (S,) int, -1 padded
    x: np.ndarray         # (S,) float, aligned with support
    resid: float
    n_iter: int
    status: int


@dataclass
class Verdict:
    outcome: str
    detail: str = ""
    coef_err: float = 0.0
    res_err: float = 0.0


def _values_ok(g: GpuSignal, o, N: int):
    k = int(g.n_iter)
    xd_g = np.zeros(N)
    if k > 0:
        xd_g[np.asarray(g.support[:k], dtype=np.int64)] = np.asarray(g.x[:k], dtype=np.float64)
    xd_o = o.dense(N)
    no = float(np.linalg.norm(xd_o))
    if no == 0.0:
        cerr = 0.0 if not np.any(xd_g) else float("inf")
    else:
        cerr = float(np.linalg.norm(xd_g - xd_o) / no)
    rerr = abs(float(g.resid) - o.resid_norm)
    rtol = RES_RTOL * o.resid_norm + RES_ATOL_Y * o.y_norm
    ok = cerr <= COEF_RTOL and rerr <= rtol
    return ok, cerr, rerr / max(o.y_norm, 1e-300)


def compare_signal(g: GpuSignal, o, N: int) -> Verdict:
    if o.status == NAN_STATUS:
        return Verdict("exact") if g.status == NAN_STATUS else Verdict("bug", "oracle NAN, gpu not")
    k_o = o.n_iter
    k_g = int(g.n_iter)
    sup_o = [int(v) for v in o.support]
    sup_g = [int(v) for v in g.support[:k_g]]
    # padding must be -1 after n_iter
    if np.any(np.asarray(g.support[k_g:]) != -1):
        return Verdict("bug", "support not -1 padded after n_iter")
    same_seq = sup_g == sup_o and k_g == k_o and int(g.status) == int(o.status)
    f = o.first_flag(extended=False)
    fe = o.first_flag(extended=True)
    if same_seq:
        ok, ce, re = _values_ok(g, o, N)
        if ok:
            return Verdict("exact" if f is None else "flagged_ok", coef_err=ce, res_err=re)
        return Verdict("bug", f"values off: coef {ce:.3g} resid {re:.3g}", ce, re)
    # first diverging decision (selection index or stop decision)
    j = 0
    while j < min(len(sup_g), len(sup_o)) and sup_g[j] == sup_o[j]:
        j += 1
    if f is not None and f <= j:
        if set(sup_g) == set(sup_o) and k_g == k_o:
            ok, ce, re = _values_ok(g, o, N)
            if ok:
                return Verdict("flagged_ok", coef_err=ce, res_err=re)
            return Verdict("bug", f"flagged, same set, values off: coef {ce:.3g} resid {re:.3g}", ce, re)
        return Verdict("tie_divergent", f"flag at {f}, diverge at {j}")
    if fe is not None and fe <= j:
        return Verdict("explained", f"extended flag at {fe}, diverge at {j}")
    return Verdict("bug", f"unflagged divergence at step {j}: gpu {sup_g[j:j+3]} ora {sup_o[j:j+3]} "
                          f"(n_iter {k_g}/{k_o}, status {g.status}/{o.status})")


@dataclass
class Report:
    counts: Counter = field(default_factory=Counter)
    bugs: List[str] = field(default_factory=list)
    max_coef_err: float = 0.0
    max_res_err: float = 0.0

    def as_dict(self) -> Dict:
        return dict(counts=dict(self.counts), bugs=self.bugs[:10], max_coef_err=self.max_coef_err,
                    max_res_err_over_ynorm=self.max_res_err)


def compare_batch(support, X, resid, n_iter, status, oracle_results: Sequence, N: int,
                  rows: Optional[Sequence[int]] = None) -> Report:
    rep = Report()
    rows = range(len(oracle_results)) if rows is None else rows
    for o, b in zip(oracle_results, rows):
        g = GpuSignal(np.asarray(support[b]), np.asarray(X[b]), float(resid[b]), int(n_iter[b]),
                      int(status[b]))
        v = compare_signal(g, o, N)
        rep.counts[v.outcome] += 1
        rep.max_coef_err = max(rep.max_coef_err, v.coef_err)
        rep.max_res_err = max(rep.max_res_err, v.res_err)
        if v.outcome == "bug":
            rep.bugs.append(f"signal {b}: {v.detail}")
    return rep
