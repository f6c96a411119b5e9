"""Batch-sharded multi-GPU driver pieces.

The method has no exchange step: every image is an independent problem, so
the batch is split across ranks and each rank runs the whole layer stack on
its images (one process per GPU, torch.distributed for the plumbing).  The
only collectives are at setup — one broadcast of each layer's stretched CSR
(rowptr/colidx/value) and bias from rank 0, over NCCL/NVLink — and after
measurement (MAX of per-rank device times).  No per-layer collectives.

These functions are device-agnostic (the tensors' device decides: CUDA
tensors with the nccl backend on the GPU box, CPU tensors with gloo in the
tests).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n_total: int, rank: int, world_size: int):
    """Contiguous image range [a, b) of `rank` (sizes differ by at most one)."""
    base, rem = divmod(n_total, world_size)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


def broadcast_csr(rowptr, colidx, value, bias, device, src: int = 0):
    """Broadcast one layer's stretched CSR + bias from `src` to every rank.

    On src the numpy arrays are given; elsewhere pass None.  Returns device
    tensors (rowptr int32, colidx int32, value fp32, bias fp32) on every rank.
    """
    rank = dist.get_rank()
    if rank == src:
        meta = torch.tensor([rowptr.size, colidx.size, bias.size], dtype=torch.int64, device=device)
    else:
        meta = torch.zeros(3, dtype=torch.int64, device=device)
    dist.broadcast(meta, src)
    nr, nnz, nb = (int(v) for v in meta.tolist())
    if rank == src:
        t = [torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in (rowptr, colidx, value, bias)]
    else:
        t = [torch.empty(nr, dtype=torch.int32, device=device), torch.empty(nnz, dtype=torch.int32, device=device),
             torch.empty(nnz, dtype=torch.float32, device=device), torch.empty(nb, dtype=torch.float32, device=device)]
    for x in t:
        if x.numel():
            dist.broadcast(x, src)
    return t


def max_over_ranks(value: float, device) -> float:
    """MAX of a per-rank scalar (device-timed milliseconds) across ranks."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
