"""Batch-sharded OMP over a torch.distributed process group (one process per GPU).

The batch shards naturally: signals are independent and A is read-only (BJ north_star: "A is broadcast
once over NVLink via NCCL, each GPU solves its slice of Y, and results are gathered at the end").

    res = omp_batch_distributed(A, Y, S, eps)   # A, Y meaningful on rank 0; result on rank 0, None elsewhere

Collectives (NCCL on GPUs, gloo on CPU): one broadcast of the problem header and of A, one scatter of
the contiguous Y slices (padded to ceil(B/W) rows), and one gather of each compact output.  There is no
per-iteration communication.  The per-rank solve is the library's own GPU path unless a `solver` is
injected (the CPU tests inject one; the product never does).
"""

from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from .omp import OMP, OMPResult


def shard_bounds(B: int, world: int, rank: int):
    """Contiguous shard of rank `rank`: rows [lo, hi) with ceil(B / world) rows per rank."""
    per = -(-B // world) if world > 0 else B
    lo = min(B, rank * per)
    hi = min(B, lo + per)
    return lo, hi, per


def _gpu_solver(mode: str):
    def solve(A, Ys, S, eps):
        with OMP(A, mode=mode) as h:
            r = h.batch(Ys, S, eps)
            torch.cuda.synchronize(A.device)
        return r
    return solve


def omp_batch_distributed(A: Optional[torch.Tensor], Y: Optional[torch.Tensor], S: int,
                          eps: Optional[float] = None, mode: str = "bf16", group=None,
                          solver: Optional[Callable] = None, device=None) -> Optional[OMPResult]:
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    # problem header: M, N, B
    hdr = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == 0:
        hdr[0], hdr[1] = A.shape
        hdr[2] = Y.shape[0]
    dist.broadcast(hdr, src=0, group=group)
    M, N, B = (int(v) for v in hdr.tolist())
    # A: once, from rank 0
    A_l = A.to(device=device, dtype=torch.float32).contiguous() if rank == 0 else \
        torch.empty((M, N), dtype=torch.float32, device=device)
    dist.broadcast(A_l, src=0, group=group)
    # Y: contiguous slices, padded to `per` rows so scatter sees equal shapes
    lo, hi, per = shard_bounds(B, world, rank)
    Y_l = torch.empty((per, M), dtype=torch.float32, device=device)
    chunks = None
    if rank == 0:
        Yd = Y.to(device=device, dtype=torch.float32)
        chunks = []
        for r in range(world):
            a, b, _ = shard_bounds(B, world, r)
            c = torch.zeros((per, M), dtype=torch.float32, device=device)
            c[: b - a] = Yd[a:b]
            chunks.append(c)
    dist.scatter(Y_l, chunks, src=0, group=group)
    n_mine = hi - lo
    solve = solver or _gpu_solver(mode)
    if n_mine > 0:
        res = solve(A_l, Y_l[:n_mine], S, eps)
    else:
        res = None
    # gather each compact output, padded to `per` rows
    outs = []
    shapes = [((per, S), torch.float32), ((per, S), torch.int32), ((per,), torch.float32),
              ((per,), torch.int32), ((per,), torch.int32)]
    fields = ("X", "support", "resid_norm", "n_iter", "status")
    for (shape, dt), name in zip(shapes, fields):
        buf = torch.zeros(shape, dtype=dt, device=device)
        if res is not None:
            buf[:n_mine] = getattr(res, name).to(device=device, dtype=dt)
        gl = [torch.empty(shape, dtype=dt, device=device) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, gl, dst=0, group=group)
        if rank == 0:
            parts = []
            for r in range(world):
                a, b, _ = shard_bounds(B, world, r)
                parts.append(gl[r][: b - a])
            outs.append(torch.cat(parts, 0))
    return OMPResult(*outs) if rank == 0 else None
