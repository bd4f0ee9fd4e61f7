"""Seeded problem generator (SURVEY.md §8(d) "Synthetic inputs").

Recipe (the paper's benchmark shape, "A in R^{8M x M}, y = R^{100 x M},
S = M/4", read as M measurements x N atoms, SURVEY §8(c) ambiguity 13; and the
configs of BASELINE.json):

* Dictionary: A_ij ~ N(0,1) i.i.d. in FP64 from ``numpy.random.default_rng([seed, 0])``;
  every column is scaled to unit Euclidean norm in FP64, then the matrix is cast
  to FP32.  (Normalising columns is input preparation, "We assume
  that A has normalized columns".)
* Signal b uses its own stream ``default_rng([seed, 1, b])`` and draws, in order:
  the true sparsity s (only when a range is configured), a support uniform
  without replacement, s coefficients N(0,1), and M noise values sigma*N(0,1)
  (only when sigma > 0).  y_b = A32 x_b + noise is formed in FP64 from the
  FP32-rounded A and then cast to FP32.
* Per-signal streams make signal b identical for every batch size and every
  shard (the batch-invariance pin P8).

Nothing here performs a step of OMP; the same FP32 arrays are handed to the
CUDA path and to the FP64 oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple, Union

import numpy as np

Sparsity = Union[int, Tuple[int, int]]

# BASELINE.json "configs", restated concretely.
CONFIGS = {
    "tiny": dict(M=32, N=64, S=4, B=16, sparsity=4, sigma=0.0, eps=None, seed=1),
    "c2": dict(M=256, N=1024, S=32, B=1000, sparsity=32, sigma=0.0, eps=None, seed=2),
    # c3: "additive noise and eps-based early stopping"; sigma=0.01, eps=sigma*sqrt(M)
    # (SURVEY §8(c) ambiguity 17 / DESIGN.md reading R17).
    "c3": dict(M=1024, N=4096, S=64, B=10000, sparsity=(16, 64), sigma=0.01,
               eps=0.01 * math.sqrt(1024), seed=3),
    "c4": dict(M=2048, N=8192, S=128, B=100000, sparsity=128, sigma=0.0, eps=None, seed=4),
    # c5: batch-size sweep B = 1 .. 1e6 (nested prefixes of one stream)
    "c5": dict(M=512, N=2048, S=50, B=1000000, sparsity=50, sigma=0.0, eps=None, seed=5),
    # the paper's Yale shape: A in R^{8064 x 1207}, 1207 signals, S = 30 -- tall (M > N),
    # where the projection path (algorithm v0) is the cheaper formulation; synthetic 30-sparse signals
    "yale": dict(M=8064, N=1207, S=30, B=1207, sparsity=30, sigma=0.0, eps=None, seed=6),
    # the paper's synthetic sweep (App. B Table 2 rows 9-10): N = 8M atoms, S = M/4, B = 100
    # (reading R13: M measurements); S-sparse noiseless signals
    "t2m1024": dict(M=1024, N=8192, S=256, B=100, sparsity=256, sigma=0.0, eps=None, seed=7),
    "t2m2048": dict(M=2048, N=16384, S=512, B=100, sparsity=512, sigma=0.0, eps=None, seed=8),
}
C5_SWEEP = (1, 10, 100, 1000, 10000, 100000, 1000000)


def config(name: str, **overrides) -> dict:
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    cfg["name"] = name
    return cfg


def make_dictionary(M: int, N: int, seed: int) -> np.ndarray:
    """Return the FP32 dictionary A, shape (M, N), unit-norm columns (norms taken in FP64)."""
    rng = np.random.default_rng([seed, 0])
    A = rng.standard_normal((M, N))
    A /= np.sqrt(np.sum(A * A, axis=0, keepdims=True))
    return A.astype(np.float32)


@dataclass
class Truth:
    supports: list = field(default_factory=list)   # list of int arrays (generation order)
    coefs: list = field(default_factory=list)      # list of float64 arrays


def _draw_signal(b: int, seed: int, N: int, M: int, sparsity: Sparsity, sigma: float):
    rng = np.random.default_rng([seed, 1, int(b)])
    if isinstance(sparsity, (tuple, list)):
        s = int(rng.integers(int(sparsity[0]), int(sparsity[1]) + 1))
    else:
        s = int(sparsity)
    supp = rng.choice(N, s, replace=False)
    coef = rng.standard_normal(s)
    noise = sigma * rng.standard_normal(M) if sigma > 0 else None
    return supp, coef, noise


def make_signals(A32: np.ndarray, indices: Sequence[int], seed: int, sparsity: Sparsity,
                 sigma: float = 0.0, with_truth: bool = False, device=None):
    """Signals y_b for the given signal indices, as an FP32 array of shape (len(indices), M).

    ``device`` (e.g. "cuda:0") forms the FP64 sums y = A x + noise with torch on that
    device instead of numpy (same draws, FP64 either way; only the summation order of
    the FP64 sum differs, which can move an FP32-rounded entry by one ulp).  Used for
    the 1e5-1e6-signal configs, where the numpy gather would take minutes.
    """
    M, N = A32.shape
    idx = np.asarray(indices, dtype=np.int64)
    draws = [_draw_signal(int(b), seed, N, M, sparsity, sigma) for b in idx]
    truth = None
    if with_truth:
        truth = Truth([d[0] for d in draws], [d[1] for d in draws])
    if device is None:
        AT64 = np.ascontiguousarray(A32.T, dtype=np.float64)  # atom rows, FP64 copy of the FP32 values
        Y = np.empty((idx.size, M), dtype=np.float32)
        for i, (supp, coef, noise) in enumerate(draws):
            y = coef @ AT64[supp]
            if noise is not None:
                y = y + noise
            Y[i] = y.astype(np.float32)
    else:
        Y = _signals_torch(A32, draws, M, device)
    return (Y, truth) if with_truth else Y


def _signals_torch(A32, draws, M, device, chunk=512):
    import torch
    AT64 = torch.from_numpy(np.ascontiguousarray(A32.T)).to(device=device, dtype=torch.float64)
    B = len(draws)
    smax = max((len(d[0]) for d in draws), default=0)
    supp = np.zeros((B, smax), np.int64)
    coef = np.zeros((B, smax), np.float64)      # zero-padded coefficients add exact zeros
    noise = np.zeros((B, M), np.float64) if any(d[2] is not None for d in draws) else None
    for i, (s, c, nz) in enumerate(draws):
        supp[i, :len(s)] = s
        coef[i, :len(c)] = c
        if nz is not None:
            noise[i] = nz
    out = np.empty((B, M), np.float32)
    for a in range(0, B, chunk):
        e = min(B, a + chunk)
        sp = torch.from_numpy(supp[a:e]).to(device)
        cf = torch.from_numpy(coef[a:e]).to(device)
        y = torch.bmm(cf[:, None, :], AT64[sp])[:, 0, :]
        if noise is not None:
            y = y + torch.from_numpy(noise[a:e]).to(device)
        out[a:e] = y.to(torch.float32).cpu().numpy()
    return out


@dataclass
class Problem:
    name: str
    A: np.ndarray            # (M, N) float32, unit-norm columns
    Y: np.ndarray            # (B, M) float32, signal-major ("y batched in the first dimension")
    S: int
    eps: Optional[float]
    seed: int
    indices: np.ndarray      # global signal ids of the rows of Y
    truth: Optional[Truth] = None

    @property
    def M(self) -> int:
        return self.A.shape[0]

    @property
    def N(self) -> int:
        return self.A.shape[1]

    @property
    def B(self) -> int:
        return self.Y.shape[0]


def make_problem(name: str, B: Optional[int] = None, indices: Optional[Sequence[int]] = None,
                 with_truth: bool = False, device=None, **overrides) -> Problem:
    cfg = config(name, **overrides)
    if indices is None:
        indices = np.arange(cfg["B"] if B is None else B)
    A = make_dictionary(cfg["M"], cfg["N"], cfg["seed"])
    out = make_signals(A, indices, cfg["seed"], cfg["sparsity"], cfg["sigma"], with_truth=with_truth,
                       device=device)
    Y, truth = out if with_truth else (out, None)
    return Problem(name=name, A=A, Y=Y, S=cfg["S"], eps=cfg["eps"], seed=cfg["seed"],
                   indices=np.asarray(indices, dtype=np.int64), truth=truth)
