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
