"""Batch-sharded OMP over a torch.distributed process group (one process per GPU).

The batch shards naturally: signals are independent and A is read-only (BJ north_star: "A is broadcast
once over NVLink via NCCL, each GPU solves its slice of Y, and results are gathered at the end";
SURVEY §8(e)).  Two forms:

    d = DistributedOMP(A, mode="bf16")         # A meaningful on rank 0: broadcast once, per-rank handle
    res = d.batch(Y, S, eps)                   # Y on rank 0 -> scatter, solve, gather -> result on rank 0
    res = omp_batch_distributed(A, Y, S, eps)  # one-shot: DistributedOMP(A).batch(Y, S, eps)

Collectives (NCCL on GPUs, gloo on CPU): per dictionary, one broadcast of the header (M, N) and of A;
per batch, one broadcast of (B, S), one scatter of the contiguous Y slices (ceil(B/W) rows each; only
a ragged last slice is padded) and ONE gather of the packed compact outputs (X, support, ||r||, n_iter,
status as 2S + 3 four-byte words per signal).  There is no per-iteration communication: each rank runs
the library's whole S-iteration solve on its slice.  Everything is enqueued on the current stream, so
a caller can time the span with CUDA events.  The per-rank solve is the library's own GPU path unless
a `solver` is injected (the CPU tests inject one; the product never does).
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


def pack_result(res: Optional[OMPResult], rows: int, S: int, device) -> torch.Tensor:
    """(rows, 2S + 3) int32 words: X bits | support | ||r|| bits | n_iter | status (zeros past res)."""
    buf = torch.zeros((rows, 2 * S + 3), dtype=torch.int32, device=device)
    if res is not None:
        n = res.X.shape[0]
        buf[:n, :S] = res.X.to(device=device, dtype=torch.float32).view(torch.int32)
        buf[:n, S:2 * S] = res.support.to(device=device, dtype=torch.int32)
        buf[:n, 2 * S] = res.resid_norm.to(device=device, dtype=torch.float32).view(torch.int32)
        buf[:n, 2 * S + 1] = res.n_iter.to(device=device, dtype=torch.int32)
        buf[:n, 2 * S + 2] = res.status.to(device=device, dtype=torch.int32)
    return buf


def unpack_result(buf: torch.Tensor, S: int) -> OMPResult:
    return OMPResult(buf[:, :S].contiguous().view(torch.float32), buf[:, S:2 * S].contiguous(),
                     buf[:, 2 * S].contiguous().view(torch.float32), buf[:, 2 * S + 1].contiguous(),
                     buf[:, 2 * S + 2].contiguous())


class DistributedOMP:
    """A dictionary bound to every rank of a process group: broadcast once, one library handle per rank."""

    def __init__(self, A: Optional[torch.Tensor], mode: str = "bf16", group=None, solver: Optional[Callable] = None,
                 device=None):
        """device: where the solve runs (default: the current CUDA device; CPU with an injected solver
        and no GPU).  Collectives run on that device with NCCL, on host copies with gloo."""
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) \
                if (solver is None or backend == "nccl") else torch.device("cpu")
        self.device = torch.device(device)
        self.comm = self.device if backend == "nccl" else torch.device("cpu")
        hdr = torch.zeros(2, dtype=torch.int64, device=self.comm)
        if self.rank == 0:
            hdr[0], hdr[1] = A.shape
        dist.broadcast(hdr, src=0, group=group)
        self.M, self.N = (int(v) for v in hdr.tolist())
        A_l = A.to(device=self.comm, dtype=torch.float32).contiguous() if self.rank == 0 else \
            torch.empty((self.M, self.N), dtype=torch.float32, device=self.comm)
        dist.broadcast(A_l, src=0, group=group)          # once per dictionary
        self.A = A_l.to(self.device)
        self.solver = solver
        self.handle = OMP(self.A, mode=mode) if solver is None else None

    def close(self):
        if self.handle is not None:
            self.handle.close()
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def batch(self, Y: Optional[torch.Tensor], S: int, eps: Optional[float] = None) -> Optional[OMPResult]:
        """Y (B, M) on rank 0 (ignored elsewhere); returns the whole batch's result on rank 0, None elsewhere."""
        dev, comm, world, rank, g = self.device, self.comm, self.world, self.rank, self.group
        hdr = torch.zeros(2, dtype=torch.int64, device=comm)
        if rank == 0:
            hdr[0], hdr[1] = Y.shape[0], S
        dist.broadcast(hdr, src=0, group=g)
        B, S = (int(v) for v in hdr.tolist())
        lo, hi, per = shard_bounds(B, world, rank)
        n_mine = hi - lo
        Y_l = torch.empty((per, self.M), dtype=torch.float32, device=comm)
        chunks = None
        if rank == 0:
            Yd = Y.to(device=comm, dtype=torch.float32)
            chunks = []
            for r in range(world):
                a, b, _ = shard_bounds(B, world, r)
                if b - a == per:
                    chunks.append(Yd[a:b].contiguous())          # a view when Y is contiguous
                else:                                           # a ragged (or empty) last slice
                    c = torch.zeros((per, self.M), dtype=torch.float32, device=comm)
                    c[: b - a] = Yd[a:b]
                    chunks.append(c)
        if world > 1:
            dist.scatter(Y_l, chunks, src=0, group=g)
        else:
            Y_l = chunks[0]
        Y_l = Y_l[:n_mine].to(dev)
        res = None
        if n_mine > 0:
            res = self.solver(self.A, Y_l, S, eps) if self.solver else self.handle.batch(Y_l, S, eps)
        buf = pack_result(res, per, S, comm)
        if world == 1:
            return unpack_result(buf[:B], S)
        gl = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, gl, dst=0, group=g)
        if rank != 0:
            return None
        parts = []
        for r in range(world):
            a, b, _ = shard_bounds(B, world, r)
            parts.append(gl[r][: b - a])
        return unpack_result(torch.cat(parts, 0), S)


def omp_batch_distributed(A: Optional[torch.Tensor], Y: Optional[torch.Tensor], S: int,
                          eps: Optional[float] = None, mode: str = "bf16", group=None,
                          solver: Optional[Callable] = None, device=None) -> Optional[OMPResult]:
    """One-shot: broadcast A, scatter Y, solve each slice, gather the results to rank 0."""
    with DistributedOMP(A, mode=mode, group=group, solver=solver, device=device) as d:
        return d.batch(Y, S, eps)
