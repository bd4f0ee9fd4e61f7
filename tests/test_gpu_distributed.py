"""The NCCL sharded driver on one GPU (world size 1): same bits as the direct call."""

import numpy as np
import pytest

from synth import make_problem

pytestmark = pytest.mark.gpu


def test_nccl_world1_matches_direct_call():
    import socket

    import torch
    import torch.distributed as dist
    from paper_2407_06434_b200 import OMP
    from paper_2407_06434_b200.distributed import omp_batch_distributed

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        prob = make_problem("c2", B=300)
        A = torch.from_numpy(prob.A).cuda()
        Y = torch.from_numpy(prob.Y).cuda()
        res = omp_batch_distributed(A, Y, prob.S)
        with OMP(A) as h:
            ref = h.batch(Y, prob.S)
            torch.cuda.synchronize()
            for k in ("X", "support", "resid_norm", "n_iter", "status"):
                assert np.array_equal(getattr(res, k).cpu().numpy(), getattr(ref, k).cpu().numpy()), k
    finally:
        dist.destroy_process_group()


def _nccl_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist
    from paper_2407_06434_b200.distributed import DistributedOMP
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        prob = make_problem("c3", B=1001)                       # ragged: 501 + 500 rows at 2 ranks
        A = torch.from_numpy(prob.A).cuda() if rank == 0 else None
        Y = torch.from_numpy(prob.Y).cuda() if rank == 0 else None
        with DistributedOMP(A) as d:
            for _ in range(2):                                   # dictionary broadcast once, two batches
                res = d.batch(Y, prob.S, float(np.float32(prob.eps)))
            torch.cuda.synchronize()
        if rank == 0:
            q.put({k: getattr(res, k).cpu().numpy() for k in ("X", "support", "resid_norm", "n_iter", "status")})
        else:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_nccl_two_gpus_bitwise_equal_to_one_gpu():
    """SURVEY §8(e) verification: per-signal results are bitwise equal across rank counts -- the batch
    scattered over 2 GPUs over NCCL, gathered on rank 0, vs one GPU (skipped with fewer than 2 GPUs)."""
    import socket

    import torch
    import torch.multiprocessing as mp
    from paper_2407_06434_b200 import OMP
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dist_res = [g for g in got if g is not None]
    assert len(dist_res) == 1
    prob = make_problem("c3", B=1001)
    with OMP(torch.from_numpy(prob.A).cuda()) as h:
        ref = h.batch(torch.from_numpy(prob.Y).cuda(), prob.S, float(np.float32(prob.eps)))
        torch.cuda.synchronize()
        for k in ("X", "support", "resid_norm", "n_iter", "status"):
            assert np.array_equal(dist_res[0][k], getattr(ref, k).cpu().numpy()), k
