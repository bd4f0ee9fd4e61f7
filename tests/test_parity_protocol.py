"""Host-side tests of the parity comparator and the synthetic generator (no GPU)."""

import numpy as np

from oracle import omp, omp_batch
from parity import GpuSignal, compare_batch, compare_signal
from synth import CONFIGS, make_dictionary, make_problem, make_signals


def _as_gpu(o, S, x_scale=1.0):
    sup = -np.ones(S, np.int64)
    x = np.zeros(S, np.float32)
    sup[:o.n_iter] = o.support
    x[:o.n_iter] = o.x * x_scale
    return GpuSignal(sup, x, o.resid_norm, o.n_iter, o.status)


def test_comparator_accepts_oracle_and_rejects_perturbations():
    prob = make_problem("c2", B=4)
    outs = omp_batch(prob.A, prob.Y, 16, workers=1)
    for o in outs:
        assert compare_signal(_as_gpu(o, 16), o, prob.N).outcome in ("exact", "flagged_ok")
        assert compare_signal(_as_gpu(o, 16, 1 + 5e-4), o, prob.N).outcome == "bug"
        g = _as_gpu(o, 16)
        g.support[[2, 3]] = g.support[[3, 2]]       # swapped selection order
        g.x[[2, 3]] = g.x[[3, 2]]
        v = compare_signal(g, o, prob.N)
        assert v.outcome in ("bug", "explained", "tie_divergent")
        g = _as_gpu(o, 16)
        g.n_iter -= 1
        g.support[g.n_iter] = -1
        assert compare_signal(g, o, prob.N).outcome != "exact"
        g = _as_gpu(o, 16)
        g.resid = o.resid_norm + 1e-3 * o.y_norm
        assert compare_signal(g, o, prob.N).outcome == "bug"


def test_compare_batch_counts():
    prob = make_problem("tiny")
    outs = omp_batch(prob.A, prob.Y, prob.S, workers=1)
    S = prob.S
    sup = np.stack([_as_gpu(o, S).support for o in outs])
    X = np.stack([_as_gpu(o, S).x for o in outs])
    rep = compare_batch(sup, X, [o.resid_norm for o in outs], [o.n_iter for o in outs],
                        [o.status for o in outs], outs, prob.N)
    assert rep.counts["bug"] == 0 and sum(rep.counts.values()) == prob.B


def test_generator_contract():
    A = make_dictionary(64, 128, 9)
    assert A.dtype == np.float32 and A.shape == (64, 128)
    np.testing.assert_allclose(np.linalg.norm(A.astype(float), axis=0), 1.0, atol=1e-6)
    assert np.array_equal(A, make_dictionary(64, 128, 9))
    Y1 = make_signals(A, [0, 1, 2, 3], 9, 5)
    Y2 = make_signals(A, [2, 3], 9, 5)
    assert np.array_equal(Y1[2:], Y2)              # per-signal streams: shard invariant
    Yn, truth = make_signals(A, [0, 1], 9, (3, 6), sigma=0.1, with_truth=True)
    assert all(3 <= len(s) <= 6 for s in truth.supports)
    assert set(CONFIGS) == {"tiny", "c2", "c3", "c4", "c5", "yale", "t2m1024", "t2m2048"}
    p = make_problem("c3", B=3)
    assert p.eps is not None and abs(p.eps - 0.32) < 1e-12 and p.Y.shape == (3, 1024)


def test_generator_torch_backend_matches_numpy():
    A = make_dictionary(64, 256, 3)
    Yn = make_signals(A, range(20), 3, (4, 9), sigma=0.01)
    Yt = make_signals(A, range(20), 3, (4, 9), sigma=0.01, device="cpu")
    np.testing.assert_allclose(Yt, Yn, rtol=2e-7, atol=1e-7)
