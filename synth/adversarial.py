"""Structured adversarial inputs for the tensor-core screen's window.

Input construction only: nothing here performs a step of OMP.  The inputs are built so that
round-to-nearest into bf16 (8-bit significand, unit roundoff 2^-8) errs as far as it can in
opposite directions on two nearly tied atoms:

* atom 0 lives on rows [0, H), atom 1 on rows [H, 2H) (orthogonal supports, random signs);
* every nonzero entry of atom 0 (and of the signal on its rows) is a power of two 2^e plus just
  under half a bf16 spacing, 2^e (1 + 2^-8 (1 - d)) with d ~ 0.01 .. 0.05, so it rounds down by
  almost 2^-8 relative (the most round-to-nearest can err, at the start of a binade);
* every entry of atom 1 (and of the signal on its rows) sits just ABOVE one, so it rounds up;
* y = (1 + eta) a_0 + a_1 with unit-norm atoms, so the true normalised correlations are
  t_0 = 1 + eta > t_1 = 1 -- a gap eta = 2e-5 relative, outside the oracle's near-tie flags
  (1e-5 t_1, extended 1e-5 t_1 + 2e-6 ||y|| = 1.3e-5) and far above FP32 rounding (~1e-6).

The screen then sees atom 1 ahead of atom 0 by about 4 x 2^-8 t / ||y|| ~ 0.011 ||r||: inside
the rigorous window 2 (c0 + c0') 1.25 ||r|| ~ 0.0196 ||r|| with c0 = 2^-7 + ..., outside the
window that an erroneous c0 = 2^-8 + ... (unit roundoff 2^-9) gives, 0.0098 ||r||.
"""

from __future__ import annotations

import numpy as np

_U = 2.0 ** -8          # bf16 unit roundoff: half the spacing at the start of a binade


def _atom(H: int, rng, direction: int, d_lo: float = 0.01, d_hi: float = 0.05):
    """H entries (some zero) of a unit-norm vector, each nonzero entry 2^e (1 + 2^-8 (1 + direction d))
    with one common d in [d_lo, d_hi]: a power of two plus just under (direction -1) or just over (+1)
    half a bf16 spacing, i.e. the largest relative rounding error bf16 round-to-nearest can make.
    Unit norm: P = sum 4^-e must equal 1 / (1 + 2^-8 (1 + direction d))^2."""
    lo_f, hi_f = 1.0 + _U * (1 + direction * d_lo), 1.0 + _U * (1 + direction * d_hi)
    band = sorted((1.0 / lo_f ** 2, 1.0 / hi_f ** 2))
    mid = 0.5 * (band[0] + band[1])
    # P = v 4^-9 for an integer v in the band; the fewest powers of four 4^-e (e >= 1) summing to it are
    # v's base-4 digits (the top one, e = 1, taking v // 4^8 copies)
    unit = 4.0 ** -9
    cands = []
    for v in range(int(np.ceil(band[0] / unit)), int(np.floor(band[1] / unit)) + 1):
        exps, rest = [1] * (v // 4 ** 8), v % 4 ** 8
        for e in range(2, 10):
            digit, rest = divmod(rest, 4 ** (9 - e))
            exps += [e] * digit
        if len(exps) <= H:
            cands.append(exps)
    if cands:
        exps = cands[int(rng.integers(len(cands)))]
        f = 1.0 / np.sqrt(float(np.sum(4.0 ** -np.asarray(exps, dtype=float))))   # 1 + 2^-8 (1 + dir d)
        d = direction * ((f - 1.0) / _U - 1.0)
        vals = np.zeros(H)
        vals[:len(exps)] = 2.0 ** -np.asarray(exps, dtype=float) * f
        return rng.permutation(vals), d
    raise RuntimeError("no power-of-two assignment found")


def make_screen_adversary(M: int, seed: int, swap: bool = False):
    """(A (M x 2) float32, y (M,) float32, eta): the FP32 argmax is atom 0 (atom 1 if swap), the
    bf16 screen errs towards the other atom.  Rows are used in two halves of H = M // 2 (M >= 48)."""
    rng = np.random.default_rng([seed, 77])
    H = M // 2
    # atom 0 rounds down, atom 1 rounds up; the signal's rows of atom 0 are scaled by 1 + eta, which
    # stays below the rounding midpoint (margin 2^-8 d >= 3.9e-5 relative > 2 eta)
    a0, _ = _atom(H, rng, -1)
    a1, _ = _atom(H, rng, +1)
    eta = 2e-5
    s0 = rng.choice([-1.0, 1.0], size=H)
    s1 = rng.choice([-1.0, 1.0], size=H)
    A = np.zeros((M, 2))
    A[:H, 0] = s0 * a0
    A[H:2 * H, 1] = s1 * a1
    y = np.zeros(M)
    y[:H] = (1.0 + eta) * A[:H, 0]
    y[H:2 * H] = A[H:2 * H, 1]
    perm = rng.permutation(M)              # scatter the rows (rounding is per entry)
    A, y = A[perm], y[perm]
    if swap:                               # the winner at index 1: lowest-index tie rules cannot help
        A = A[:, ::-1]
    return A.astype(np.float32), y.astype(np.float32), eta
