"""Image sharding across GPUs: one process per GPU, no collective on the data path.

The BNN path partitions perfectly by image (no reduction crosses images,
SURVEY section 8(e)), so N ranks take contiguous image ranges, run the whole
fused plan independently, and only int32 logits / predictions are gathered
(40 B per image).  torch.distributed (NCCL on the box, gloo in the CPU
tests) is used for the barrier, the max-over-ranks timing reduction and the
optional result gather -- plumbing, not the product.
"""

from __future__ import annotations

import os

import numpy as np


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process = (0, 1, 0))."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_bounds(n: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) image range of ``rank``; sizes differ by at most one."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} of {world_size}")
    base, extra = divmod(int(n), world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def init(backend: str | None = None):
    """Initialise the default process group when launched under torchrun (no-op otherwise)."""
    import torch
    import torch.distributed as dist

    rank, ws, local = world()
    if ws == 1 or dist.is_initialized():
        return
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=ws, device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend, rank=rank, world_size=ws)


def barrier():
    import torch.distributed as dist

    if dist.is_initialized():
        dist.barrier()


def max_over_ranks(value: float) -> float:
    """Max of a scalar across ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_results(logits: np.ndarray, preds: np.ndarray, n_total: int, dst: int = 0):
    """Assemble every rank's (logits, preds) shard on rank ``dst`` in image order.

    Returns (logits (n_total, classes), preds (n_total,)) on ``dst`` and None elsewhere.
    Off the timed path: runs once after the benchmark / inference.
    """
    import torch.distributed as dist

    if not dist.is_initialized():
        return logits, preds
    rank, ws = dist.get_rank(), dist.get_world_size()
    parts = [None] * ws if rank == dst else None
    dist.gather_object((np.asarray(logits), np.asarray(preds)), parts, dst=dst)
    if rank != dst:
        return None
    all_l = np.concatenate([p[0] for p in parts])
    all_p = np.concatenate([p[1] for p in parts])
    assert all_l.shape[0] == n_total, (all_l.shape, n_total)
    return all_l, all_p


def sharded_infer(engine, model, images: np.ndarray, gather: bool = True):
    """Each rank runs its contiguous shard of ``images`` through ``engine``; gathers on rank 0."""
    rank, ws, _ = world()
    lo, hi = shard_bounds(images.shape[0], ws, rank)
    logits, preds = engine.infer(model, images[lo:hi])
    if not gather:
        return logits, np.asarray(preds)
    return gather_results(logits, np.asarray(preds), images.shape[0])
