"""Multi-GPU plumbing for the hot path (one process per GPU).

SURVEY.md §8(e): the decode path shards by request with no data-path
collective — each rank owns its requests' KV pool, summaries, tables and
selections (``KVStore``) — so the only cross-rank operations are the
measurement barriers and the max-over-ranks of the timed region.  The
KV-head-sharded configuration (config 5) splits the KV heads of every layer
over a head group and all-gathers the attention outputs after each layer
(``HeadGroup``, one NCCL all-gather over NVLink inside the step graph;
DESIGN.md §6).  tests/test_gpu_dist.py runs it as 2 ranks on one GPU (gloo)
against the 1-rank engine, bit for bit.
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


# ---------------------------------------------------------------------------
# KV-head-sharded decode (config 5, SURVEY.md §8e option (i)):
# the world is split into `n_head_shards`-rank head groups (each rank owns
# H / n_head_shards KV heads of every layer) x `n_replicas` request replicas
# (each replica group owns B / n_replicas request rows).  After each layer's
# attention the head group all-gathers its outputs over NVLink — the path's
# only exchange step; no softmax merge is needed because a query head's
# attention is entirely local to the rank owning its KV head.

def head_shard_layout(world: int, n_kv_heads: int) -> tuple[int, int]:
    """(n_head_shards, n_replicas): the largest head split that divides both
    the world and the KV heads; the rest of the world replicates requests."""
    shards = 1
    for s in range(1, world + 1):
        if world % s == 0 and n_kv_heads % s == 0:
            shards = s
    return shards, world // shards


def head_shard_of(rank: int, world: int, n_kv_heads: int, batch: int):
    """This rank's (kv head range, request rows, head-group ranks)."""
    shards, replicas = head_shard_layout(world, n_kv_heads)
    replica, shard = divmod(rank, shards)
    per = n_kv_heads // shards
    heads = range(shard * per, (shard + 1) * per)
    rows = shard_rows(batch, replica, replicas)
    group = [replica * shards + s for s in range(shards)]
    return heads, rows, group


class HeadGroup:
    """All-gather of per-shard attention outputs [B_r, Hq/shards, d] into the
    full [B_r, Hq, d] (query heads in KV-head order) within a head group."""

    def __init__(self, world: int, n_kv_heads: int):
        self.shards, self.replicas = head_shard_layout(world, n_kv_heads)
        self.group = None
        if dist.is_initialized() and self.shards > 1:
            groups = [dist.new_group([r * self.shards + s for s in range(self.shards)])
                      for r in range(self.replicas)]  # every rank creates every group
            self.group = groups[dist.get_rank() // self.shards]

    def gather(self, local: torch.Tensor, out: torch.Tensor) -> None:
        """local [B_r, Hq/shards, d] -> out [B_r, Hq, d]."""
        if self.group is None:
            out.copy_(local)
            return
        local = local.contiguous()
        if dist.get_backend(self.group) == "nccl":  # one NCCL all-gather over NVLink
            stacked = torch.empty((self.shards,) + tuple(local.shape), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(stacked, local, group=self.group)
        else:  # gloo (CPU tests)
            parts = [torch.empty_like(local) for _ in range(self.shards)]
            dist.all_gather(parts, local, group=self.group)
            stacked = torch.stack(parts)
        out.copy_(stacked.permute(1, 0, 2, 3).reshape(out.shape))
