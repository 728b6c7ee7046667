"""Book sharding across GPUs (one process per GPU, torch.distributed).

Books are independent, so the path shards with no
communication: rank r owns a contiguous range of GLOBAL book ids, and the seeded
generator keys every stream by its global id, so a book's bytes -- and hence its
outputs -- are identical at every world size.  The only collectives run after
the timed region: the max of the per-rank elapsed times and a gather of the
per-book counters (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_books(rank: int, world: int, books: int, scaling: str = "weak") -> tuple[int, int]:
    """(first global book id, number of books) owned by `rank`.

    weak:   every rank owns `books` books (global ids rank*books ...);
    strong: `books` is the total, split into contiguous near-equal ranges.
    """
    if world < 1 or not 0 <= rank < world or books < 0:
        raise ValueError("bad rank/world/books")
    if scaling == "weak":
        return rank * books, books
    if scaling == "strong":
        base, extra = divmod(books, world)
        begin = rank * base + min(rank, extra)
        return begin, base + (1 if rank < extra else 0)
    raise ValueError(f"unknown scaling {scaling!r}")


def _active():
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def _coll_device(device):
    """NCCL reduces device tensors; gloo (CPU tests, single-GPU multi-rank checks) host tensors."""
    return device if dist.get_backend() == "nccl" else "cpu"


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (the timing rule: a multi-GPU time is the slowest rank's)."""
    if not _active():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: int, device=None) -> int:
    if not _active():
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=_coll_device(device))
    dist.all_reduce(t)
    return int(t.item())


def gather_rows(local: torch.Tensor) -> torch.Tensor:
    """Concatenate every rank's [n_i, ...] tensor in rank order (variable n_i allowed)."""
    if not _active():
        return local
    if dist.get_backend() != "nccl" and local.is_cuda:
        return gather_rows(local.cpu()).to(local.device)
    world = dist.get_world_size()
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    if dist.get_backend() == "nccl":
        out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, pad)
        parts = out.split(m)
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])
