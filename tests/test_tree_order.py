"""Host check of a summation-order identity the update kernel relies on (update_core.cuh, z = F^T w).

With F_k in shared memory a thread sums column j itself instead of a warp: it forms the 32 lane partials
and adds them as the adjacent-pair tree over the leaves in bit-reversed order.  The claim is that this is,
bit for bit, the value lane 0 holds after the warp's xor tree `acc += shfl_xor(acc, o)`, o = 16 .. 1
(IEEE addition is commutative, and level o pairs lanes l and l ^ o).  Emulated here in float32.
"""

import numpy as np


def xor_tree_lane0(p):
    acc = p.astype(np.float32).copy()
    for o in (16, 8, 4, 2, 1):
        acc = (acc + acc[np.arange(32) ^ o]).astype(np.float32)
    assert np.all(acc.view(np.uint32) == acc[0].view(np.uint32))   # every lane ends with the same bits
    return acc[0]


def brev_adjacent_tree(p):
    brev = [int(f"{r:05b}"[::-1], 2) for r in range(32)]
    q = [np.float32(p[brev[r]]) for r in range(32)]
    h = 1
    while h < 32:
        for r in range(0, 32, 2 * h):
            q[r] = np.float32(q[r] + q[r + h])
        h *= 2
    return q[0]


def test_bit_reversed_adjacent_tree_equals_warp_xor_tree():
    rng = np.random.default_rng(7)
    for trial in range(2000):
        scale = 10.0 ** rng.integers(-8, 8, size=32)
        p = (rng.standard_normal(32) * scale).astype(np.float32)
        if trial % 5 == 0:
            p[rng.integers(0, 32, size=rng.integers(1, 31))] = 0.0   # columns shorter than 32 rows
        if trial % 7 == 0:
            p[rng.integers(0, 32)] = -0.0
        a, b = xor_tree_lane0(p), brev_adjacent_tree(p)
        assert a.view(np.uint32) == b.view(np.uint32), (trial, a, b)


def test_a_different_pairing_is_not_bitwise_equal():
    """The check above can fail: sequential left-to-right summation differs on the same inputs."""
    rng = np.random.default_rng(8)
    diff = 0
    for _ in range(200):
        p = (rng.standard_normal(32) * 10.0 ** rng.integers(-4, 4, size=32)).astype(np.float32)
        s = np.float32(0)
        for v in p:
            s = np.float32(s + v)
        diff += int(s.view(np.uint32) != xor_tree_lane0(p).view(np.uint32))
    assert diff > 50
