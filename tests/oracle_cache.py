"""On-disk cache of FP64 oracle results for the survey-sized parity samples (SURVEY §8(d) table
"Oracle / parity subsample") -- TEST INFRASTRUCTURE.

The cache is written by ``scripts/build_oracle_cache.py``, which calls only ``synth`` (the seeded
inputs) and ``oracle`` (the FP64 Algorithm 1).  Each entry is keyed by (config, seed, signal index)
and carries a hash of the signal's FP32 bytes: a GPU-side generator may form y in another FP64
summation order and move an entry by one ulp, and such a signal is then recomputed by the oracle on
the spot instead of being compared against a result for a different input.

Stored per signal: what tests/parity.py compares (support, x, ||r||, n_iter, status, ||y||) and the
first flagged step under the primary and the extended near-tie rules (-1 = none), plus which kinds
of flag the signal carries (for the report's flag counts).
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE_DIR = os.path.join(HERE, "golden", "oracle_cache")

C4_SHARD_ROWS = np.array(sorted({b for r in range(8) for b in
                                 list(range(r * 12500, r * 12500 + 64)) +
                                 list(range((r + 1) * 12500 - 64, (r + 1) * 12500))}), dtype=np.int64)
# the samples: c4 1 024 signals = 64 at each end of every rank's slice at 8 GPUs (which
# contains the 1-, 2- and 4-GPU boundaries); c3 2 000 of 10 000; c5 1 000 of B = 10^6
SAMPLES = {
    "c4": C4_SHARD_ROWS,
    "c3": np.arange(0, 10000, 5, dtype=np.int64),
    "c5": np.linspace(0, 999999, 1000).astype(np.int64),
}


def y_hash(y32: np.ndarray) -> int:
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(y32, dtype=np.float32).tobytes(),
                                          digest_size=8).digest(), "little")


@dataclass
class CachedResult:
    """The fields of oracle.OracleResult that tests/parity.py reads."""
    support: np.ndarray
    x: np.ndarray
    resid_norm: float
    n_iter: int
    status: int
    y_norm: float
    ff_primary: int
    ff_extended: int
    flags: Dict[str, bool]

    def dense(self, N: int) -> np.ndarray:
        out = np.zeros(N)
        out[self.support] = self.x
        return out

    def first_flag(self, extended: bool = False) -> Optional[int]:
        f = self.ff_extended if extended else self.ff_primary
        return None if f < 0 else int(f)


def summarize(o) -> dict:
    """The flag kinds of one oracle result (any step)."""
    return dict(primary=any(s.primary_tie for s in o.steps),
                extended=any(s.extended_tie for s in o.steps),
                stop=bool(o.init_stop_flag) or any(s.stop_flag for s in o.steps),
                near_degenerate=any(s.near_degenerate for s in o.steps))


def cache_path(name: str) -> str:
    return os.path.join(CACHE_DIR, f"{name}.npz")


def save(name: str, seed: int, S: int, eps, indices: Sequence[int], Y: np.ndarray, results) -> str:
    n = len(results)
    sup = -np.ones((n, S), np.int32)
    x = np.zeros((n, S), np.float64)
    fields = {k: np.zeros(n, bool) for k in ("primary", "extended", "stop", "near_degenerate")}
    ffp = -np.ones(n, np.int32)
    ffe = -np.ones(n, np.int32)
    for i, o in enumerate(results):
        sup[i, :o.n_iter] = o.support
        x[i, :o.n_iter] = o.x
        f = o.first_flag(False)
        fe = o.first_flag(True)
        ffp[i] = -1 if f is None else f
        ffe[i] = -1 if fe is None else fe
        for k, v in summarize(o).items():
            fields[k][i] = v
    os.makedirs(CACHE_DIR, exist_ok=True)
    path = cache_path(name)
    np.savez_compressed(path, seed=seed, S=S, eps=np.nan if eps is None else eps,
                        indices=np.asarray(indices, np.int64),
                        yhash=np.array([y_hash(y) for y in Y], dtype=np.uint64),
                        support=sup, x=x, resid_norm=np.array([o.resid_norm for o in results]),
                        y_norm=np.array([o.y_norm for o in results]),
                        n_iter=np.array([o.n_iter for o in results], np.int32),
                        status=np.array([o.status for o in results], np.int32),
                        ff_primary=ffp, ff_extended=ffe,
                        **{f"flag_{k}": v for k, v in fields.items()})
    return path


def load(name: str):
    """{signal index: (y hash, CachedResult)} or None if the cache file is absent."""
    path = cache_path(name)
    if not os.path.exists(path):
        return None
    z = np.load(path)
    out = {}
    for i, b in enumerate(z["indices"]):
        k = int(z["n_iter"][i])
        out[int(b)] = (int(z["yhash"][i]), CachedResult(
            support=z["support"][i, :k].astype(np.int64), x=z["x"][i, :k].copy(),
            resid_norm=float(z["resid_norm"][i]), n_iter=k, status=int(z["status"][i]),
            y_norm=float(z["y_norm"][i]), ff_primary=int(z["ff_primary"][i]),
            ff_extended=int(z["ff_extended"][i]),
            flags={f: bool(z[f"flag_{f}"][i]) for f in ("primary", "extended", "stop", "near_degenerate")}))
    return out


def oracle_for_rows(name: str, A: np.ndarray, Y: np.ndarray, rows: Sequence[int], indices: Sequence[int],
                    S: int, eps, workers=None):
    """Oracle results for rows `rows` of Y (global signal ids `indices[rows]`): from the cache when the
    signal's FP32 bytes match, else computed now.  Returns (results, n_from_cache)."""
    from oracle import omp_batch
    cache = load(name) or {}
    res = [None] * len(rows)
    todo = []
    for j, r in enumerate(rows):
        hit = cache.get(int(indices[r]))
        if hit is not None and hit[0] == y_hash(Y[r]):
            res[j] = hit[1]
        else:
            todo.append(j)
    if todo:
        fresh = omp_batch(A, Y[[rows[j] for j in todo]], S, eps, workers=workers)
        for j, o in zip(todo, fresh):
            res[j] = o
    return res, len(rows) - len(todo)
