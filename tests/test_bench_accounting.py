"""Host logic of bench.py's roofline accounting (no GPU): the algorithmic work per launch follows the
signals each launch actually processes (SURVEY §8(d) per-unit figures x live signals)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import config  # noqa: E402


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_runs_equal_the_default_accounting(name):
    cfg = config(name)
    B = 1000
    w0 = bench.kernel_work(cfg, B, "bf16", "residual")
    w1 = bench.kernel_work(cfg, B, "bf16", "residual", np.full(B, cfg["S"]))
    for k in ("correlation", "update", "select"):
        assert w1[k][1] == pytest.approx(w0[k][1], rel=1e-12), k
    # 2 M N flops per signal-iteration for the screen
    assert w0["correlation"][1] == pytest.approx(2.0 * cfg["M"] * cfg["N"] * B)


def test_early_stops_reduce_the_work():
    cfg = config("c3")
    S, B = cfg["S"], 1000
    n_iter = np.full(B, S)
    n_iter[: B // 2] = S // 2            # half the batch stops at S/2 (eps)
    w = bench.kernel_work(cfg, B, "bf16", "residual", n_iter)
    full = bench.kernel_work(cfg, B, "bf16", "residual")
    assert w["correlation"][1] == pytest.approx(0.75 * full["correlation"][1])
    assert w["update"][1] < full["update"][1]
    # signals stopped at k = 0 (eps >= ||y||) cost nothing
    none = bench.kernel_work(cfg, B, "bf16", "residual", np.zeros(B, dtype=np.int32))
    assert none["correlation"][1] == 0.0 and none["update"][1] == 0.0


def test_update_bytes_split():
    """update = streamed (HBM) + gathered (L2) bytes; the gather is (k + 2) atom rows of 4 Mp bytes."""
    cfg = config("c4")
    S, M = cfg["S"], cfg["M"]
    bound, total, unit, split = bench.kernel_work(cfg, 1, "bf16", "residual")["update"]
    assert bound == "l2" and unit == "GB/s"
    assert total == pytest.approx(split["hbm_bytes"] + split["l2_gather_bytes"])
    ks = np.arange(S)
    assert split["l2_gather_bytes"] == pytest.approx(float((4.0 * M * (ks + 2)).sum() / S))


def test_update_streamed_bytes_count_every_screen_partial():
    """The screen writes TOPK = 4 (value, index) float2 per 128-atom group (Np / 128 groups), and the update
    reads all of them: 8 x 4 x Np / 128 bytes per signal-iteration (round 1 counted per 256-atom tile)."""
    cfg = config("c4")
    S, M, N = cfg["S"], cfg["M"], cfg["N"]
    Mp = -(-M // 64) * 64
    ks = np.arange(S, dtype=np.float64)
    hbm = bench.kernel_work(cfg, 1, "bf16", "residual")["update"][3]["hbm_bytes"]
    want = (4.0 * Mp + 8.0 * 4 * (N // 128) + 4.0 * ks * (ks + 1) / 2 + 4.0 * (ks + 2) * 3 + 4.0 * M
            + (4.0 + 2.0) * Mp).sum() / S
    assert hbm == pytest.approx(want)
