"""The tensor-core screen's window against adversarially rounded inputs -- CPU only.

The bf16 screen computes sum_m bf16(a_m / ||a||) bf16(r_m) in FP32; round-to-nearest into bf16
(8-bit significand) errs by up to 2^-8 relative per operand, so the screen may be off by up to
(2^-7 + 2^-16) ||r|| per normalised correlation, and the FP32 argmax is guaranteed to be among the
candidates only if the window covers twice that.  `synth.adversarial` builds two nearly tied atoms
whose operands sit just below / just above bf16 rounding midpoints; here the screen's arithmetic is
emulated exactly in numpy (the products of two bf16 values are exact, the 2 x 64-term sums are
far inside FP32) and checked against the library's own window (ompScreeningWindow, host code).
"""

import numpy as np
import pytest

from oracle import omp
from synth.adversarial import make_screen_adversary

CASES = [(M, seed, swap) for M in (48, 64, 256, 1024) for seed in (0, 1) for swap in (False, True)]


def bf16_rn(x):
    """float32 -> nearest bf16 (ties to even), returned as float64."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def emulated_screen(A32, y32):
    """|c~_n| of the bf16 screen: atoms normalised in FP32 as the setup kernel does (1/||a|| from an
    FP64 norm), both operands rounded to bf16, exact products summed (FP32 accumulation error of
    <= 64 x 2^-23 relative on these all-positive products is far below the effect tested)."""
    ss = np.sum(A32.astype(np.float64) ** 2, axis=0)
    inv = (1.0 / np.sqrt(ss)).astype(np.float32)
    ahat = (A32 * inv[None, :]).astype(np.float32)
    return np.abs(bf16_rn(ahat).T @ bf16_rn(y32))


@pytest.fixture(scope="module")
def window():
    from paper_2407_06434_b200 import build
    from paper_2407_06434_b200.omp import screening_window
    build.build()
    return screening_window


def old_window(M):
    """The round-1 window: c0 = 2^-8 + 2^-18 + Kp 2^-23 (it took bf16's unit roundoff as 2^-9)."""
    Kp = -(-M // 64) * 64
    c0 = 2.0 ** -8 + 2.0 ** -18 + Kp * 2.0 ** -23
    return 2.5 * (c0 + (Kp / 32 + 8) * 2.0 ** -23)


@pytest.mark.parametrize("M,seed,swap", CASES)
def test_adversary_defeats_the_round1_window_not_the_rigorous_one(window, M, seed, swap):
    A, y, eta = make_screen_adversary(M, seed, swap)
    win, lose = (1, 0) if swap else (0, 1)
    # the FP64 oracle: the winner is selected with a clear, unflagged gap
    o = omp(A, y, 2)
    assert list(o.support) == [win, lose]
    st = o.steps[0]
    assert not st.primary_tie and not st.extended_tie
    assert (st.t1 - st.t2) / st.t1 > 1.5e-5
    # the emulated screen puts the loser ahead by more than the round-1 window ...
    v = emulated_screen(A, y)
    rn = float(np.linalg.norm(y.astype(np.float64)))
    lead = (v[lose] - v[win]) / rn
    assert lead > old_window(M), (lead, old_window(M))
    # ... and by less than the library's window, which therefore keeps the FP32 argmax a candidate
    W = window("bf16", M)
    assert lead < W, (lead, W)
    # and every screened value is within the per-element bound c0 = W / 2.5 - c0'
    Kp = -(-M // 64) * 64
    c0 = W / 2.5 - (Kp / 32 + 8) * 2.0 ** -23
    exact = np.abs(A.astype(np.float64).T @ y.astype(np.float64)) / np.linalg.norm(A.astype(np.float64), axis=0)
    assert np.max(np.abs(v - exact)) / rn <= c0


def test_library_window_values(window):
    """The window's constants, and -1 where there is no screen."""
    for M in (32, 256, 2048, 8192):
        Kp = -(-M // 64) * 64
        bf = 2.5 * (2.0 ** -7 + 2.0 ** -16 + 2.0 ** -22 + Kp * 2.0 ** -23 + (Kp / 32 + 8) * 2.0 ** -23)
        x3 = 2.5 * (2.0 ** -20 + 2.0 ** -22 + 3 * Kp * 2.0 ** -23 + (Kp / 32 + 8) * 2.0 ** -23)
        assert window("bf16", M) == pytest.approx(bf, rel=1e-6)
        assert window("3xtf32", M) == pytest.approx(x3, rel=1e-6)
        assert window("simt", M) == -1.0


def adaptive_window(A32, y32, M):
    """The per-signal window the library uses in bf16 mode (WinCoef):
    W = 2.5 (E_a (|r| + d) + d + K 2^-23 (1 + E_a)(|r| + d) + c0' |r|), E_a = max_n |bf16(a_n/|a_n|) - a_n/|a_n||,
    d = |r - bf16(r)| -- both measured on the actual operands (here emulated exactly)."""
    A64 = A32.astype(np.float64)
    ss = np.sum(A64 ** 2, axis=0)
    inv = (1.0 / np.sqrt(ss)).astype(np.float32)
    ahat32 = (A32 * inv[None, :]).astype(np.float32)
    Ea = np.max(np.linalg.norm(bf16_rn(ahat32) - A64 / np.sqrt(ss)[None, :], axis=0))
    r = y32.astype(np.float64)
    rn = np.linalg.norm(r)
    d = np.linalg.norm(r - bf16_rn(y32))
    Kp = -(-M // 64) * 64
    u = 2.0 ** -23
    return 2.5 * (Ea * (rn + d) + d + Kp * u * (1 + Ea) * (rn + d) + (Kp / 32 + 8) * u * rn), Ea, d / rn


@pytest.mark.parametrize("M,seed,swap", CASES)
def test_adaptive_window_covers_the_adversary(window, M, seed, swap):
    """The measured-rounding window widens on adversarial operands (E_a, d/|r| near 2^-8) and still
    covers the screen's lead; it never exceeds the static worst case (ompScreeningWindow)."""
    A, y, _ = make_screen_adversary(M, seed, swap)
    win, lose = (1, 0) if swap else (0, 1)
    v = emulated_screen(A, y)
    rn = float(np.linalg.norm(y.astype(np.float64)))
    lead = (v[lose] - v[win]) / rn
    W, Ea, drel = adaptive_window(A, y, M)
    assert Ea > 0.9 * 2.0 ** -8 and drel > 0.9 * 2.0 ** -8      # the operands err almost maximally
    assert lead < W / rn <= window("bf16", M) * (1 + 1e-6)


def test_adaptive_window_is_narrower_on_gaussian_data(window):
    """On the configs' Gaussian data the measured rounding is ~2.3x below the worst case, so the
    per-signal window is about half the static bound (fewer FP32 re-evaluations)."""
    from synth import make_problem
    prob = make_problem("c2", B=8)
    for y in prob.Y:
        W, Ea, drel = adaptive_window(prob.A, y, prob.M)
        rn = float(np.linalg.norm(y.astype(np.float64)))
        assert 0.3 < (W / rn) / window("bf16", prob.M) < 0.6
