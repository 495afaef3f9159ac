"""Multi-GPU plumbing for the hot path (one process per GPU).

SURVEY.md §8(e): the decode path shards by request with no data-path
collective — each rank owns its requests' KV pool, summaries, tables and
selections (``KVStore``) — so the only cross-rank operations are the
measurement barriers and the max-over-ranks of the timed region.  The
KV-head-sharded configuration (one all-gather of attention outputs per layer)
is listed as next work in DESIGN.md §6.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from torchrun's environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Initialise the default process group when WORLD_SIZE > 1 (NCCL on GPU,
    gloo on CPU) and bind this process to its GPU."""
    rank, world, local = env_rank()
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return rank, world, local


def shard_rows(total: int, rank: int, world: int) -> range:
    """Request rows owned by ``rank`` when ``total`` requests are split
    request-parallel (contiguous, sizes differ by at most one)."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(x: float) -> float:
    """Max of a scalar over all ranks (the timed region's slowest rank)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
