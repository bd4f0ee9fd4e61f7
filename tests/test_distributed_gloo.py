"""World-size-2 gloo tests of the batch-sharded driver's host logic (no GPU).

The per-rank solve is injected: an FP64-oracle solver stands in for the GPU path here (tests may use
the oracle; the product never does).  What is tested is the sharding, the collectives and the gather:
the distributed result must equal the single-process oracle result signal by signal.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_solver(A, Ys, S, eps):
    from oracle import omp_batch
    from paper_2407_06434_b200.omp import OMPResult
    out = omp_batch(A.numpy(), Ys.numpy(), S, eps, workers=1)
    n = len(out)
    X = torch.zeros((n, S), dtype=torch.float32)
    sup = torch.full((n, S), -1, dtype=torch.int32)
    for i, o in enumerate(out):
        X[i, :o.n_iter] = torch.from_numpy(o.x.astype(np.float32))
        sup[i, :o.n_iter] = torch.from_numpy(o.support.astype(np.int32))
    return OMPResult(X, sup, torch.tensor([o.resid_norm for o in out], dtype=torch.float32),
                     torch.tensor([o.n_iter for o in out], dtype=torch.int32),
                     torch.tensor([o.status for o in out], dtype=torch.int32))


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_06434_b200.distributed import omp_batch_distributed
        from synth import make_problem
        prob = make_problem("tiny", B=B, sigma=0.02)
        A = torch.from_numpy(prob.A) if rank == 0 else None
        Y = torch.from_numpy(prob.Y) if rank == 0 else None
        res = omp_batch_distributed(A, Y, prob.S, None, solver=oracle_solver)
        if rank == 0:
            q.put({k: getattr(res, k).numpy() for k in ("X", "support", "resid_norm", "n_iter", "status")})
        else:
            q.put(None if res is None else "non-root got a result")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [16, 7, 1])
def test_sharded_equals_single_process(B):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from synth import make_problem
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    root = [g for g in got if isinstance(g, dict)]
    assert len(root) == 1 and all(g is None for g in got if not isinstance(g, dict))
    res = root[0]
    prob = make_problem("tiny", B=B, sigma=0.02)
    ref = oracle_solver(torch.from_numpy(prob.A), torch.from_numpy(prob.Y), prob.S, None)
    assert np.array_equal(res["support"], ref.support.numpy())
    assert np.array_equal(res["X"], ref.X.numpy())
    assert np.array_equal(res["n_iter"], ref.n_iter.numpy())


def test_shard_bounds_cover_the_batch():
    from paper_2407_06434_b200.distributed import shard_bounds
    for B in (1, 7, 16, 100000):
        for W in (1, 2, 3, 8):
            rows = []
            for r in range(W):
                lo, hi, per = shard_bounds(B, W, r)
                assert 0 <= hi - lo <= per
                rows.extend(range(lo, hi))
            assert rows == list(range(B))


def _worker_persistent(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_06434_b200.distributed import DistributedOMP
        from synth import make_problem
        prob = make_problem("tiny", B=11, sigma=0.02)
        A = torch.from_numpy(prob.A) if rank == 0 else None
        outs = []
        with DistributedOMP(A, solver=oracle_solver) as d:
            assert (d.M, d.N) == prob.A.shape
            for B in (11, 4, 3):                       # several batches on one broadcast dictionary
                Y = torch.from_numpy(prob.Y[:B]) if rank == 0 else None
                r = d.batch(Y, prob.S if B != 3 else 2)
                outs.append(None if r is None else {k: getattr(r, k).numpy() for k in
                                                    ("X", "support", "resid_norm", "n_iter", "status")})
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


def test_distributed_handle_serves_several_batches():
    """DistributedOMP: A broadcast once, then batches of different B (ragged, and B < world x 2) and S,
    each scattered, solved per rank and gathered to rank 0 (ONE packed gather per batch)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from synth import make_problem
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_persistent, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o is None for o in got[1])
    prob = make_problem("tiny", B=11, sigma=0.02)
    for (B, S), res in zip(((11, prob.S), (4, prob.S), (3, 2)), got[0]):
        ref = oracle_solver(torch.from_numpy(prob.A), torch.from_numpy(prob.Y[:B]), S, None)
        for k in ("X", "support", "resid_norm", "n_iter", "status"):
            assert np.array_equal(res[k], getattr(ref, k).numpy()), (B, k)


def test_pack_unpack_round_trip():
    from paper_2407_06434_b200.distributed import pack_result, unpack_result
    from paper_2407_06434_b200.omp import OMPResult
    rng = np.random.default_rng(3)
    S, n = 5, 7
    r = OMPResult(torch.from_numpy(rng.standard_normal((n, S)).astype(np.float32)),
                  torch.from_numpy(rng.integers(-1, 100, (n, S)).astype(np.int32)),
                  torch.tensor([np.nan, 1.5, -0.0, 3, 4, 5, 6], dtype=torch.float32),
                  torch.arange(n, dtype=torch.int32), torch.arange(n, dtype=torch.int32) % 4)
    u = unpack_result(pack_result(r, n + 2, S, torch.device("cpu"))[:n], S)
    for k in ("X", "support", "resid_norm", "n_iter", "status"):
        a, b = getattr(r, k), getattr(u, k)
        assert a.dtype == b.dtype and torch.equal(a.view(torch.int32) if a.is_floating_point() else a,
                                                  b.view(torch.int32) if b.is_floating_point() else b), k
