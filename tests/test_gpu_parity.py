"""GPU parity: the CUDA path (through the C ABI) vs the FP64 oracle on the same seeded inputs.

Protocol and tolerances: tests/parity.py (BASELINE.json north_star):
supports bit-exact outside oracle-flagged near-ties, coefficients <= 1e-4 relative L2,
residual norms <= 1e-4 relative (+1e-5 ||y|| floor, reading R10).
"""

import json
import os

import numpy as np
import pytest

from gpu_helpers import assert_no_bugs, eps32, parity, parity_cached, run_gpu
from oracle_cache import SAMPLES
from oracle import DEGENERATE, EPS, MAXITER, NAN
from synth import make_dictionary, make_problem, make_signals

pytestmark = pytest.mark.gpu
MODES = ["bf16", "3xtf32", "simt", "small", "proj"]   # gpu_helpers.PATHS ("small" = persistent kernel,
                                                     # "proj" = projection path / algorithm v0)
LIB_MODES = ["bf16", "3xtf32", "simt"]
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
STATUS = {"MAXITER": MAXITER, "EPS": EPS, "DEGENERATE": DEGENERATE, "NAN": NAN}


# ------------------------------------------------------------------ correlation GEMM (K1)
def screening_bound(mode, K):
    """Rigorous |c~ - c| / (||a|| ||r||) of each correlation kernel: operand rounding
    (bf16: round-to-nearest, unit roundoff 2^-8 per operand -> 2^-7 + 2^-16, plus 2^-22 for the FP32
    normalisation of the atom; 3xTF32: tf32-truncated lo terms + dropped lo*lo) plus at most one
    truncation of the FP32 accumulator per product (K, or 3K for the three 3xTF32 products) x 2^-23."""
    Kp = -(-K // 64) * 64
    if mode == "bf16":
        return 2.0 ** -7 + 2.0 ** -16 + 2.0 ** -22 + Kp * 2.0 ** -23
    if mode == "3xtf32":
        return 2.0 ** -20 + 2.0 ** -22 + 3 * Kp * 2.0 ** -23
    return 1e-6


@pytest.mark.parametrize("mode", LIB_MODES)
@pytest.mark.parametrize("shape", [(32, 64, 16), (256, 1024, 1000), (300, 700, 333), (1024, 4096, 520),
                                   (2048, 8192, 1024)])
def test_correlation_gemm_vs_fp64(mode, shape):
    """K1 numerics: SIMT is FP32-accurate; the tensor-core screens stay inside their rigorous bound."""
    import torch
    from paper_2407_06434_b200 import OMP
    M, N, B = shape
    rng = np.random.default_rng(M + N + B)
    A = rng.standard_normal((M, N)).astype(np.float32)
    R = rng.standard_normal((B, M)).astype(np.float32)
    with OMP(torch.from_numpy(A).cuda(), mode=mode) as h:
        C = h.correlate(torch.from_numpy(R).cuda()).cpu().numpy()
        G = h.gram().cpu().numpy()
    ref = R.astype(np.float64) @ A.astype(np.float64)
    scale = np.linalg.norm(R, axis=1)[:, None] * np.linalg.norm(A, axis=0)[None, :]
    err = np.abs(C - ref) / scale
    print(f"{mode} {shape}: max |C - C64| / (|r||a|) = {err.max():.3e}  bound {screening_bound(mode, M):.3e}")
    if mode == "simt":
        assert err.max() <= 1e-6
    else:
        # the bound is rigorous; with M >= 256 terms the rounding errors average well inside it
        assert err.max() <= screening_bound(mode, M) * (0.5 if M >= 256 else 1.0)
    A64 = A.astype(np.float64)
    Gref = A64.T @ A64
    gs = np.linalg.norm(A, axis=0)
    gerr = np.abs(G - Gref) / (gs[:, None] * gs[None, :])
    assert gerr.max() <= 1e-5   # G is FP32/round-to-nearest in every mode; diagonal = M same-sign terms


# ------------------------------------------------------------------ worked examples (P5) on the GPU
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("ex", GOLD["omp"], ids=[e["name"] for e in GOLD["omp"]])
def test_worked_examples_gpu(mode, ex):
    A = np.array(ex["A_columns"], dtype=np.float32).T.copy()
    y = np.array([ex["y"]], dtype=np.float32)
    out = run_gpu(A, y, ex["S"], ex.get("eps"), mode)
    e = ex["expect"]
    k = len(e["support"])
    assert out["status"][0] == STATUS[e["status"]]
    assert out["n_iter"][0] == k
    assert list(out["support"][0][:k]) == e["support"]
    assert np.all(out["support"][0][k:] == -1)
    np.testing.assert_allclose(out["X"][0][:k], e["x"], atol=1e-6)
    assert np.all(out["X"][0][k:] == 0)


# ------------------------------------------------------------------ configs
@pytest.mark.parametrize("mode", MODES)
def test_parity_tiny(mode):
    prob = make_problem("tiny")
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, mode)
    rep = parity(out, prob.A, prob.Y, prob.S, prob.eps, range(prob.B))
    d = assert_no_bugs(rep, f"tiny/{mode}")
    assert d["counts"].get("exact", 0) == prob.B
    # init + per-iteration kernels; init + the persistent kernel; Y planes + P0 GEMM + init + one kernel
    # per iteration + final residual
    want = {"small": 2, "proj": prob.S + 5, "simt": 1 + 3 * prob.S}.get(mode, 1 + 2 * prob.S)
    assert out["launches"] == want
    assert out["path"] == {"small": "small", "proj": "projection"}.get(mode, "residual")


@pytest.mark.parametrize("mode", LIB_MODES)
def test_parity_c2_all(mode):
    prob = make_problem("c2")
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, mode)
    rep = parity(out, prob.A, prob.Y, prob.S, prob.eps, range(prob.B))
    d = assert_no_bugs(rep, f"c2/{mode}")
    assert d["counts"].get("exact", 0) + d["counts"].get("flagged_ok", 0) >= 995


@pytest.fixture(scope="module")
def c3_problem():
    return make_problem("c3", device="cuda")


@pytest.mark.parametrize("mode", LIB_MODES)
def test_parity_c3_full_batch_sampled(mode, c3_problem):
    """c3 at its full batch (B = 10^4, eps stops): 2 000 signals (every 5th) against the oracle
    (SURVEY §8(d) subsample; cached FP64 results, tests/oracle_cache.py)."""
    prob = c3_problem
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, mode)
    rows = SAMPLES["c3"]
    assert len(rows) == 2000
    assert_no_bugs(parity_cached(out, prob, rows, "c3"), f"c3/{mode}")
    st = out["status"]
    assert np.mean(st == EPS) > 0.95            # c3 stops by eps


@pytest.mark.parametrize("B", [1, 10, 1000, 100000])
def test_parity_c5_sweep_sampled(B):
    prob = make_problem("c5", B=B, device="cuda" if B > 1000 else None)
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "auto")
    rows = np.unique(np.linspace(0, B - 1, min(B, 48)).astype(int))
    assert_no_bugs(parity(out, prob.A, prob.Y, prob.S, prob.eps, rows), f"c5 B={B}")


@pytest.fixture(scope="module")
def c4_problem():
    return make_problem("c4", device="cuda")


@pytest.mark.parametrize("mode", ["auto", "3xtf32"])
def test_parity_c4_full_batch_sampled(mode, c4_problem):
    """BASELINE.json's largest config at its full size (B = 1e5), the bench's launch configuration
    (auto = bf16 screen) and the 3xTF32 screen: the 1 024 signals at the ends of every rank's slice at
    8 GPUs (cached FP64 results), plus every signal that stopped before S."""
    prob = c4_problem
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, mode)
    odd = np.flatnonzero((out["status"] != MAXITER) | (out["n_iter"] != prob.S))
    print(f"c4/{mode}: {len(odd)} signals stopped before S: statuses {np.unique(out['status'][odd], return_counts=True)}")
    assert len(odd) <= 100
    rows = sorted(set(SAMPLES["c4"].tolist()) | set(odd[:16].tolist()))
    assert len(rows) >= 1024
    assert_no_bugs(parity_cached(out, prob, rows, "c4"), f"c4/{mode}")


def test_parity_c5_1e6_sampled():
    """c5 at B = 10^6 (the sweep's largest batch, in the bench's launch configuration): 1 000 signals
    spread over the batch against cached FP64 results."""
    prob = make_problem("c5", device="cuda")
    assert prob.B == 1000000
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "auto")
    assert_no_bugs(parity_cached(out, prob, SAMPLES["c5"], "c5"), "c5 B=1e6")


# ------------------------------------------------------------------ ragged shapes, edge cases
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("MNBS", [(33, 77, 5, 7), (100, 300, 129, 20), (257, 513, 257, 31)])
def test_ragged_shapes(mode, MNBS):
    M, N, B, S = MNBS
    A = make_dictionary(M, N, 17)
    Y = make_signals(A, range(B), 17, max(2, S // 2), sigma=0.01)
    out = run_gpu(A, Y, S, None, mode)
    assert_no_bugs(parity(out, A, Y, S, None, range(B)), f"ragged {MNBS}/{mode}")


@pytest.mark.parametrize("mode", MODES)
def test_edge_cases(mode):
    A = make_dictionary(64, 128, 5)
    A[:, 9] = A[:, 3]                       # duplicate atom -> DEGENERATE after exhaustion
    Y = make_signals(A, range(6), 5, 3)
    Y[1] = 0.0                              # zero signal: eps=0 stops at k = 0
    Y[2, 7] = np.nan                        # NaN signal
    Y[3] = 2.0 * A[:, 3] - A[:, 50]         # exactly 2-sparse with a duplicated atom
    yn = np.linalg.norm(Y[4].astype(np.float64))
    # eps >= ||y_4|| stops before the first selection; others keep going
    out = run_gpu(A, Y, 8, 0.0, mode)
    assert out["status"][1] == EPS and out["n_iter"][1] == 0 and np.all(out["support"][1] == -1)
    assert out["status"][2] == NAN and out["n_iter"][2] == 0
    # an exact 2-atom fit: the residual path's FP32 r is tiny but nonzero, so it goes on and stops
    # DEGENERATE (or at S); the projection path's ||r||^2 = ||y||^2 - ||u||^2 may cancel to exactly
    # 0 <= eps = 0 and stop by eps after the two atoms (reading R22)
    ok = (DEGENERATE, MAXITER, EPS) if mode == "proj" else (DEGENERATE, MAXITER)
    assert out["status"][3] in ok
    assert set(out["support"][3][:2]) == {3, 50}
    if out["status"][3] == EPS:
        assert out["n_iter"][3] == 2
    out = run_gpu(A, Y[4:5], 8, float(yn) * 1.0001, mode)
    assert out["status"][0] == EPS and out["n_iter"][0] == 0
    assert out["resid"][0] == pytest.approx(yn, rel=1e-6)


def test_invalid_dictionary_and_args():
    import torch
    from paper_2407_06434_b200 import OMP, OmpError
    A = make_dictionary(16, 32, 1)
    A[:, 7] = 0.0
    with pytest.raises(OmpError) as ei:
        OMP(torch.from_numpy(A).cuda())
    assert ei.value.status == 2 and ei.value.detail == 7
    A[:, 7] = 1.0
    A[3, 11] = np.inf
    with pytest.raises(OmpError) as ei:
        OMP(torch.from_numpy(A).cuda())
    assert ei.value.status == 3 and ei.value.detail == 11
    A = make_dictionary(16, 32, 1)
    with OMP(torch.from_numpy(A).cuda()) as h:
        Y = torch.zeros((3, 16), device="cuda")
        with pytest.raises(OmpError):
            h.batch(Y, 17)                   # S > M
        with pytest.raises(OmpError):
            h.batch(Y, 0)
        r = h.batch(Y[:0], 4)                # B = 0 is a no-op
        assert r.X.shape == (0, 4)


@pytest.mark.parametrize("mode", LIB_MODES)
def test_batch_invariance_bitwise(mode):
    """P8: signal b's result does not depend on B or on its position (no split-K in K1)."""
    prob = make_problem("c2", B=300)
    full = run_gpu(prob.A, prob.Y, prob.S, None, mode)
    part = run_gpu(prob.A, prob.Y[130:260], prob.S, None, mode)
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(full[key][130:260], part[key]), key


@pytest.mark.parametrize("mode", ["bf16", "3xtf32"])
def test_overflowing_screen_groups_find_the_exact_argmax(mode):
    """Many exact ties inside one 128-atom screen group (12 orthonormal atoms with equal coefficients):
    more in-window entries than the screen keeps, so the group is flagged as overflowing and the update
    must still land on the exact FP32 argmax.  The small-batch kernel evaluates every atom exactly (same
    dot order, no screen), so the two paths must agree bit for bit."""
    rng = np.random.default_rng(11)
    M = 256
    Q1 = np.linalg.qr(rng.standard_normal((M, M)))[0]
    Q2 = np.linalg.qr(rng.standard_normal((M, M)))[0]
    A = np.concatenate([Q1, Q2], axis=1).astype(np.float32)          # N = 512: four 128-atom groups
    # 12 tied atoms inside group 0; starts 58 and 62 straddle atom 64, where (K = 256 < 1536) the screen's
    # 16-warp epilogue splits the group between two warps that merge their in-window lists
    starts = (0, 3, 40, 100, 58, 62)
    Y = np.zeros((len(starts), M), dtype=np.float32)
    for b, start in enumerate(starts):
        Y[b] = A[:, start:start + 12].astype(np.float64).sum(axis=1).astype(np.float32)
    scr = run_gpu(A, Y, 12, None, mode)
    small = run_gpu(A, Y, 12, None, "small")
    assert scr["path"] == "residual" and small["path"] == "small"
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(scr[key], small[key]), key
    for b, start in enumerate(starts):                               # every tied atom is recovered
        assert set(scr["support"][b].tolist()) == set(range(start, start + 12))


ADVERSARY_CASES = [(M, seed, swap) for M in (48, 64, 256, 1024) for seed in (0, 1) for swap in (False, True)]


@pytest.mark.parametrize("mode", ["bf16", "3xtf32"])
def test_screen_window_adversarial_rounding(mode):
    """Two nearly tied atoms (FP32 gap 2e-5 relative, unflagged by the oracle) whose operands sit just
    below / just above bf16 rounding midpoints (synth.adversarial; tests/test_screen_window.py shows
    on the CPU that the bf16 screen then ranks the loser ahead by 0.0107 ||r||, more than the round-1
    window 0.0098 ||r||, less than the rigorous 0.0196 ||r||).  16 copies per signal on the screened
    path (small-batch limit 0), every decision against the oracle, bitwise against the small-batch
    kernel (exact FP32 over all atoms)."""
    from synth.adversarial import make_screen_adversary
    for M, seed, swap in ADVERSARY_CASES:
        A, y, _ = make_screen_adversary(M, seed, swap)
        Y = np.repeat(y[None, :], 16, axis=0)
        scr = run_gpu(A, Y, 2, None, mode)
        small = run_gpu(A, Y, 2, None, "small")
        assert scr["path"] == "residual" and small["path"] == "small"
        win = 1 if swap else 0
        assert np.all(scr["support"] == [win, 1 - win]), (M, seed, swap, scr["support"][0])
        for key in ("support", "X", "resid", "n_iter", "status"):
            assert np.array_equal(scr[key], small[key]), (M, seed, swap, key)
        d = assert_no_bugs(parity(scr, A, Y, 2, None, range(2)), f"adversary {M}/{seed}/{swap}/{mode}")
        assert d["counts"].get("exact", 0) == 2


@pytest.mark.parametrize("copies", [1, 16], ids=["groups", "all-N"])
@pytest.mark.parametrize("mode", ["bf16", "3xtf32"])
def test_refine_overflowing_groups_and_all_atoms(mode, copies):
    """Exact ties filling the screen's groups: the dictionary is `copies` side-by-side copies of the
    identity (M = 1024), y = the sum of 600 unit vectors, so every 128-atom group holds ~75 tied
    entries -- more than its 4 kept slots -- and is re-evaluated whole: 8 groups for one copy; 128
    groups for 16 copies, more than the 64-group list holds, so the update re-evaluates all N = 16 384
    atoms.  Exact ties -> lowest index (reading R4): the tied atoms of the first copy in ascending
    order, every coefficient exactly 1, ||r||^2 = 600 - S exactly.  Then (one copy) a random orthonormal
    dictionary with the same structure (ties to ~1e-7): bitwise equal to the small-batch kernel, which
    evaluates every atom exactly."""
    M = 1024
    N = M * copies
    S, B = 16, 16
    rng = np.random.default_rng(5)
    T = [np.sort(rng.choice(M, 600, replace=False)) for _ in range(B)]
    A = np.tile(np.eye(M, dtype=np.float32), (1, copies))
    Y = np.zeros((B, M), dtype=np.float32)
    for b in range(B):
        Y[b, T[b]] = 1.0
    scr = run_gpu(A, Y, S, None, mode)
    small = run_gpu(A, Y, S, None, "small")
    for b in range(B):
        assert np.array_equal(scr["support"][b], T[b][:S]), b
    assert np.all(scr["X"] == 1.0) and np.all(scr["status"] == MAXITER) and np.all(scr["n_iter"] == S)
    assert np.all(scr["resid"] == np.float32(np.sqrt(600 - S)))
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(scr[key], small[key]), key
    if copies > 1:
        return
    Q = np.linalg.qr(rng.standard_normal((M, M)))[0].astype(np.float32)
    Yq = np.stack([Q[:, T[b]].astype(np.float64).sum(axis=1) for b in range(B)]).astype(np.float32)
    scr = run_gpu(Q, Yq, S, None, mode)
    small = run_gpu(Q, Yq, S, None, "small")
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(scr[key], small[key]), key
    # (600-way near-ties at every step: every signal may diverge after its first flag)
    assert_no_bugs(parity(scr, Q, Yq, S, None, range(4)), f"orthonormal ties/{mode}", max_excused_frac=1.0)


@pytest.mark.parametrize("name", ["c2", "c5", "c4"])
def test_update_block_size_invariance_bitwise(name):
    """The per-iteration update picks its block size from the batch (one warp per signal for B >= 8192
    at M <= 512, wider CTAs below, a high-ILP variant when B <= 2 x SMs); every reduction of the tail
    runs in a T-independent order, so signal b's bits are the same in all of them (and with the
    programmatic-dependent-launch edge on or off).  c4 (M = 2048): the 8192-signal batch keeps F_k in
    L1 / L2 and sums z = F^T w warp per column (shuffle tree), the smaller ones stage F_k (k <= 63) in
    shared memory and sum it thread per column in the same pairing -- the same bits."""
    prob = make_problem(name, B=8192)
    big = run_gpu(prob.A, prob.Y, prob.S, None, "bf16")
    mid = run_gpu(prob.A, prob.Y[1000:3000], prob.S, None, "bf16")     # 2000 signals: wider CTAs
    few = run_gpu(prob.A, prob.Y[4000:4100], prob.S, None, "bf16")     # 100 signals: few-CTA variant
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(big[key][1000:3000], mid[key]), key
        assert np.array_equal(big[key][4000:4100], few[key]), key
    rows = range(0, 100, 7) if name != "c4" else range(0, 100, 50)
    assert_no_bugs(parity(few, prob.A, prob.Y[4000:4100], prob.S, None, rows), f"{name} B=100")


@pytest.mark.parametrize("case", [("tiny", 16, {}), ("c2", 64, {}), ("c5", 20, {}), ("c5", 64, {"eps": 0.05}),
                                  ("c3", 8, {}), ("c4", 2, {})], ids=lambda c: f"{c[0]}-B{c[1]}")
def test_small_path_bitwise_equals_screened(case):
    """The persistent small-batch kernel and the screened per-iteration path return the same bits:
    n* is the exact FP32 argmax on both (rigorous screen window), and they share the append/residual
    code (update_core.cuh).  Covers KC = 4 / 8 / 16 register tiles (M = 32 .. 2048) and eps stops."""
    name, B, over = case
    prob = make_problem(name, B=B, **over)
    small = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "small")
    scr = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "bf16")
    assert small["path"] == "small" and scr["path"] == "residual"
    assert small["launches"] == 2 and scr["launches"] == 1 + 2 * prob.S
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(small[key], scr[key]), key
    rows = range(min(B, 8))
    assert_no_bugs(parity(small, prob.A, prob.Y, prob.S, prob.eps, rows), f"small {name} B={B}")


@pytest.mark.parametrize("case", [("c2", 300, {}), ("c3", 400, {}), ("c5", 200, {}), ("yale", 96, {})],
                         ids=lambda c: f"{c[0]}-B{c[1]}")
def test_projection_path_parity(case):
    """The projection path (algorithm v0) against the oracle: selections from
    p = P0 - sum_j x_j G[s_j, :], the eps test from ||y||^2 - ||u||^2 (reading R22), exact final ||r||."""
    name, B, over = case
    prob = make_problem(name, B=B, **over)
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "proj")
    assert out["launches"] == prob.S + 5 and out["path"] == "projection"
    rows = range(B) if prob.A.shape[0] <= 1024 else range(0, B, 6)
    d = assert_no_bugs(parity(out, prob.A, prob.Y, prob.S, prob.eps, rows), f"proj {name} B={B}")
    assert d["counts"].get("exact", 0) + d["counts"].get("flagged_ok", 0) >= 0.97 * len(rows)


@pytest.mark.parametrize("name", ["t2m1024", "t2m2048"])
def test_paper_sweep_shapes_sampled(name):
    """The paper's own synthetic sweep shapes (App. B Table 2 rows 9-10: N = 8M, S = M/4, B = 100),
    full batch in the bench's launch configuration, sampled rows against the oracle."""
    prob = make_problem(name)
    out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "auto")
    rows = [0, 37, 99] if name == "t2m1024" else [0, 99]
    assert_no_bugs(parity(out, prob.A, prob.Y, prob.S, prob.eps, rows), name)


def test_auto_algorithm_picks_projection_for_tall_dictionaries():
    """Cost model: the Yale shape (M = 8064 > N = 1207) runs the projection path, c2 the residual path."""
    yale = make_problem("yale", B=16)
    assert run_gpu(yale.A, yale.Y, yale.S, None, "auto")["path"] == "projection"
    c2 = make_problem("c2", B=8)
    assert run_gpu(c2.A, c2.Y, c2.S, None, "auto")["path"] == "small"          # B <= 8
    c2b = make_problem("c2", B=100)
    assert run_gpu(c2b.A, c2b.Y, c2b.S, None, "auto")["path"] == "residual"


def _fields(r):
    return [t.cpu().numpy() for t in (r.X, r.support, r.resid_norm, r.n_iter, r.status)]


@pytest.mark.parametrize("mode", ["bf16", "simt"])
def test_graph_replay_matches_direct_launch(mode):
    """The CUDA-graph replay (default path) equals direct launches (ompSetGraphs(0)) bit for bit,
    across graph-cache hits, misses (fresh output buffers, new eps, new B) and evictions."""
    import torch
    from paper_2407_06434_b200 import OMP
    prob = make_problem("c2", B=300)
    Y = torch.from_numpy(prob.Y).cuda()
    with OMP(torch.from_numpy(prob.A).cuda(), mode=mode) as h:
        h.set_graphs(False)
        want = {}
        for B, eps in [(300, None), (300, 0.3), (77, None)]:
            r = h.batch(Y[:B], prob.S, eps)
            want[(B, eps)] = _fields(r)
        h.set_graphs(True)
        for rep in range(3):
            for (B, eps), w in want.items():
                r = h.batch(Y[:B], prob.S, eps)   # fresh outputs each call
                got = _fields(r)
                for a, b in zip(got, w):
                    assert np.array_equal(a, b), (rep, B, eps)
        assert h.launch_count() == 1 + (3 if mode == "simt" else 2) * prob.S
        for _ in range(6):                        # > cache size distinct keys: eviction path
            outs = h.batch(Y[:300], prob.S)
        assert np.array_equal(outs.support.cpu().numpy(), want[(300, None)][1])
        # profiling mode: graphs with an event node on either side of every kernel, same bits, and the
        # per-kernel times of each replay (one launch of every kernel per batch)
        h.profile(True)
        h.profile_read(reset=True)
        for rep in range(3):
            r = h.batch(Y[:300], prob.S)
            if rep == 1:
                h.profile_read(reset=False)       # read between replays; the third is collected lazily
            got = _fields(r)
            for a, b in zip(got, want[(300, None)]):
                assert np.array_equal(a, b), ("profiled", rep)
        prof = h.profile_read(reset=True)
        h.profile(False)
        assert prof["correlation"][1] == 3 * prob.S and prof["update"][1] == 3 * prob.S
        assert prof["init"][1] == 3 and prof["update"][0] > 0 and prof["correlation"][0] > 0


def test_host_path_matches_device_path():
    import torch
    from paper_2407_06434_b200 import OMP
    prob = make_problem("c2", B=200)
    with OMP(torch.from_numpy(prob.A).cuda()) as h:
        dev = h.batch(torch.from_numpy(prob.Y).cuda(), prob.S)
        host = h.batch_host(prob.Y, prob.S)
        torch.cuda.synchronize()
        assert np.array_equal(dev.support.cpu().numpy(), host.support)
        assert np.array_equal(dev.X.cpu().numpy(), host.X)
        assert np.array_equal(dev.resid_norm.cpu().numpy(), host.resid_norm)
        Xd = h.densify(dev).cpu().numpy()
    sup = host.support
    for b in range(5):
        k = host.n_iter[b]
        want = np.zeros(prob.N, np.float32)
        want[sup[b, :k]] = host.X[b, :k]
        assert np.array_equal(Xd[b], want)


@pytest.mark.parametrize("mode", ["bf16", "simt", "small", "proj"])
def test_strided_buffers_match_contiguous(mode):
    """Leading dimensions beyond the minimum (lda > M, ldy > M, ldx / lds > S) on every path give the
    same bits as contiguous buffers; nothing outside the logical rows/columns is touched."""
    import torch
    from gpu_helpers import PATHS
    from paper_2407_06434_b200 import OMP, OMPResult
    lib_mode, small, algo = PATHS[mode]
    M, N, B, S = 100, 300, 6 if mode == "small" else 40, 9
    A = make_dictionary(M, N, 21)
    Y = make_signals(A, range(B), 21, 6, sigma=0.01)
    Aw = torch.zeros((N, M + 5), dtype=torch.float32, device="cuda")   # atom n at row n: lda = M + 5
    Aw[:, :M] = torch.from_numpy(A.T.copy()).cuda()
    Yw = torch.full((B, M + 7), 7.0, dtype=torch.float32, device="cuda")
    Yw[:, :M] = torch.from_numpy(Y).cuda()

    def run(Adev, Ydev, out=None):
        with OMP(Adev, mode=lib_mode) as h:
            h.set_small_batch_limit(small)
            h.set_algorithm(algo)
            r = h.batch(Ydev, S, 0.05, out=out)
            torch.cuda.synchronize()
            assert h.last_path() == {"small": "small", "proj": "projection"}.get(mode, "residual")
            return r

    ref = run(torch.from_numpy(A).cuda(), torch.from_numpy(Y).cuda())
    Xw = torch.full((B, S + 3), -9.0, dtype=torch.float32, device="cuda")
    Sw = torch.full((B, S + 3), -9, dtype=torch.int32, device="cuda")
    out = OMPResult(Xw[:, :S], Sw[:, :S], torch.empty(B, device="cuda"),
                    torch.empty(B, dtype=torch.int32, device="cuda"), torch.empty(B, dtype=torch.int32, device="cuda"))
    got = run(Aw[:, :M].t(), Yw[:, :M], out=out)
    for key in ("X", "support", "resid_norm", "n_iter", "status"):
        assert torch.equal(getattr(ref, key), getattr(got, key)), key
    assert torch.all(Xw[:, S:] == -9.0) and torch.all(Sw[:, S:] == -9)


def test_host_path_chunked_pipeline_matches_device_path():
    """ompBatchHost splits a large batch into chunks whose copies overlap the solve; the results are
    bitwise those of one device call."""
    import torch
    from paper_2407_06434_b200 import OMP
    prob = make_problem("c5", B=140000, device="cuda")     # >= 2 x 65536: two chunks
    with OMP(torch.from_numpy(prob.A).cuda()) as h:
        dev = h.batch(torch.from_numpy(prob.Y).cuda(), prob.S)
        torch.cuda.synchronize()
        host = h.batch_host(prob.Y, prob.S)
        for key, a, b in (("support", dev.support, host.support), ("X", dev.X, host.X),
                          ("resid", dev.resid_norm, host.resid_norm), ("n_iter", dev.n_iter, host.n_iter),
                          ("status", dev.status, host.status)):
            assert np.array_equal(a.cpu().numpy(), b), key


def test_inverse_cholesky_state_identity():
    """P9 on the GPU's own factor: F_k V_k^T = I with V_k from numpy.linalg.cholesky."""
    import torch
    from paper_2407_06434_b200 import OMP
    prob = make_problem("c2", B=4)
    S = prob.S
    with OMP(torch.from_numpy(prob.A).cuda()) as h:
        res = h.batch(torch.from_numpy(prob.Y).cuda(), S)
        F, u = h.factor(0, 4, S)
        F, u = F.cpu().numpy(), u.cpu().numpy()
        sup = res.support.cpu().numpy()
    A64 = prob.A.astype(np.float64)
    for b in range(4):
        Fd = np.zeros((S, S))
        for j in range(S):
            Fd[:j + 1, j] = F[b, j * (j + 1) // 2: j * (j + 1) // 2 + j + 1]
        A_k = A64[:, sup[b]]
        V = np.linalg.cholesky(A_k.T @ A_k)
        assert np.abs(Fd @ V.T - np.eye(S)).max() <= 5e-5
        np.testing.assert_allclose(u[b], Fd.T @ (A_k.T @ prob.Y[b].astype(np.float64)), atol=2e-5)


def test_one_shot_c_abi_omp_batch():
    """The north star's one-shot call omp_batch(A, Y, S, eps) -> X, support, ||r|| through ctypes with
    device pointers (column-major A, lda = M; Y M x B, ldy = M), bitwise equal to the handle API."""
    import ctypes
    import torch
    from paper_2407_06434_b200 import _lib
    lib = _lib.load()
    prob = make_problem("c3", B=300)
    M, N, S, B = prob.M, prob.N, prob.S, prob.B
    A = torch.from_numpy(np.ascontiguousarray(prob.A.T)).cuda()     # atom n at A + n * M
    Y = torch.from_numpy(prob.Y).cuda()                               # signal b at Y + b * M
    X = torch.empty((B, S), device="cuda")
    sup = torch.empty((B, S), dtype=torch.int32, device="cuda")
    res = torch.empty(B, device="cuda")
    nit = torch.empty(B, dtype=torch.int32, device="cuda")
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.omp_batch(A.data_ptr(), M, N, Y.data_ptr(), B, S, ctypes.c_float(eps32(prob.eps)), X.data_ptr(),
                       sup.data_ptr(), res.data_ptr(), nit.data_ptr(), st.data_ptr(), stream)
    assert rc == 0
    want = run_gpu(prob.A, prob.Y, S, prob.eps, "auto")
    for key, got in (("X", X), ("support", sup), ("resid", res), ("n_iter", nit), ("status", st)):
        assert np.array_equal(got.cpu().numpy(), want[key]), key
    assert lib.omp_batch(A.data_ptr(), M, N, Y.data_ptr(), B, 0, ctypes.c_float(-1.0), X.data_ptr(), sup.data_ptr(),
                         res.data_ptr(), nit.data_ptr(), st.data_ptr(), stream) == 1     # S = 0


def test_expanded_and_overlapping_inputs_are_copied():
    """Y = y.expand(B, M) (row stride 0) must not make the library read B x M floats of a buffer that
    holds M: the binding copies such views; the result equals the contiguous batch bit for bit."""
    import torch
    from paper_2407_06434_b200 import OMP
    prob = make_problem("c2", B=1)
    with OMP(torch.from_numpy(prob.A).cuda()) as h:
        y = torch.from_numpy(prob.Y[0]).cuda()
        got = h.batch(y.expand(40, prob.M), prob.S)
        want = h.batch(y.expand(40, prob.M).contiguous(), prob.S)
        for key in ("X", "support", "resid_norm", "n_iter", "status"):
            assert torch.equal(getattr(got, key), getattr(want, key)), key
        one = h.batch(y.expand(1, prob.M), prob.S)        # B = 1: any row stride is fine
        assert torch.equal(one.support, want.support[:1])


def test_projection_needs_n_at_most_8192():
    """The projection path runs N-wide rows (N <= 8192): AUTO picks the residual path for a tall
    dictionary with N > 8192 (M = 8064, N = 9000 would favour projection), and an explicit projection
    request fails with OMP_ERR_UNSUPPORTED before any launch, leaving the handle usable."""
    import torch
    from paper_2407_06434_b200 import OMP, OmpError
    M, N, S, B = 8064, 9000, 4, 16
    A = make_dictionary(M, N, 31)
    Y = make_signals(A, range(B), 31, S)
    with OMP(torch.from_numpy(A).cuda()) as h:
        Yd = torch.from_numpy(Y).cuda()
        h.set_algorithm("projection")
        with pytest.raises(OmpError) as ei:
            h.batch(Yd, S)
        assert ei.value.status == 6
        h.set_algorithm("auto")
        r = h.batch(Yd, S)
        torch.cuda.synchronize()
        assert h.last_path() == "residual"
        out = dict(support=r.support.cpu().numpy(), X=r.X.cpu().numpy(), resid=r.resid_norm.cpu().numpy(),
                   n_iter=r.n_iter.cpu().numpy(), status=r.status.cpu().numpy())
    assert_no_bugs(parity(out, A, Y, S, None, range(4)), "N=9000 residual")


def test_persisting_l2_limit_is_restored():
    """ompCreate raises the device's persisting-L2 limit for the atom table (process state); the last
    handle on the device to be destroyed restores the caller's value (and a second handle in between
    keeps it raised)."""
    import ctypes
    import torch
    from paper_2407_06434_b200 import OMP
    torch.cuda.init()
    rt = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            rt = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if rt is None:
        pytest.skip("libcudart not loadable")
    LIMIT_PERSISTING_L2 = 0x06            # cudaLimitPersistingL2CacheSize

    def limit():
        v = ctypes.c_size_t()
        assert rt.cudaDeviceGetLimit(ctypes.byref(v), LIMIT_PERSISTING_L2) == 0
        return v.value

    assert rt.cudaDeviceSetLimit(LIMIT_PERSISTING_L2, ctypes.c_size_t(0)) == 0
    before = limit()
    A = torch.from_numpy(make_dictionary(2048, 4096, 3)).cuda()
    h1 = OMP(A)
    raised = limit()
    h2 = OMP(A)
    h1.close()
    assert limit() == raised              # h2 still holds it
    h2.close()
    assert limit() == before
    assert raised > before


_EPI_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
from gpu_helpers import run_gpu
from synth import make_problem
prob = make_problem(sys.argv[2], B=int(sys.argv[3]))
out = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "bf16")
np.savez(sys.argv[4], **{k: out[k] for k in ("support", "X", "resid", "n_iter", "status")})
"""


@pytest.mark.parametrize("name,B", [("c5", 300), ("c2", 257), ("c3", 200)])
def test_screen_epilogue_warp_count_bitwise(name, B, tmp_path):
    """Below K = 1536 the screen's epilogue runs on 16 warps (64 columns each, the two warps of a 128-atom
    group merging their in-window lists), above on 8.  The partial lists, hence every result, must be
    the same bits either way: compared against a process that forces the 8-warp epilogue
    (OMP_B200_EPI16_KMAX=0)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prob = make_problem(name, B=B)
    mine = run_gpu(prob.A, prob.Y, prob.S, prob.eps, "bf16")
    f = tmp_path / "epi8.npz"
    env = dict(os.environ, OMP_B200_EPI16_KMAX="0")
    subprocess.run([sys.executable, "-c", _EPI_SCRIPT, root, name, str(B), str(f)], env=env, check=True,
                   timeout=600)
    other = np.load(f)
    for key in ("support", "X", "resid", "n_iter", "status"):
        assert np.array_equal(mine[key], other[key]), key
