"""Request-parallel sharding and the max-over-ranks timing protocol, run with
world_size 2 on CPU (gloo).  The decode path has no data-path collective
(SURVEY.md §8e); these are the only cross-rank operations."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2511_00868_b200 import dist as fdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    r, w, _ = fdist.init(backend="gloo")
    rows = fdist.shard_rows(64, r, w)
    # each rank "times" a different amount; the reported value is the max
    t = fdist.max_over_ranks(1.0 + r)
    n = fdist.sum_over_ranks(len(rows))
    fdist.barrier()
    q.put((r, list(rows)[:1], len(rows), t, n))
    torch.distributed.destroy_process_group()


def test_two_rank_gloo_sharding_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, f0, n0, t0, s0), (r1, f1, n1, t1, s1) = out
    assert (f0, f1) == ([0], [32]) and n0 == n1 == 32
    assert t0 == t1 == 2.0           # max over ranks
    assert s0 == s1 == 64            # every request owned exactly once


@pytest.mark.parametrize("total,world", [(64, 2), (64, 8), (7, 3), (0, 4), (5, 8)])
def test_shard_rows_partition(total, world):
    rows = [list(fdist.shard_rows(total, r, world)) for r in range(world)]
    flat = [x for rr in rows for x in rr]
    assert flat == list(range(total))
    assert max(map(len, rows)) - min(map(len, rows)) <= 1


def _head_worker(rank, world, port, q):
    try:
        _head_body(rank, world, port, q)
    except Exception as exc:  # surface worker failures instead of a queue timeout
        q.put((rank, "error", repr(exc), None, None))


def _head_body(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    fdist.init(backend="gloo")
    H, G, D, B = 4, 7, 8, 6
    heads, rows, group = fdist.head_shard_of(rank, world, H, B)
    hg = fdist.HeadGroup(world, H)
    # each rank "computes" outputs of its query heads: value = global q-head index
    local = torch.stack([torch.full((len(heads) * G, D), 0.0)] * len(rows))
    for i, h in enumerate(heads):
        for g in range(G):
            local[:, i * G + g] = h * G + g
    out = torch.empty((len(rows), H * G, D))
    hg.gather(local, out)
    q.put((rank, list(heads), list(rows), group, out[:, :, 0].tolist()))
    torch.distributed.destroy_process_group()


def test_head_sharded_all_gather_gloo():
    """config 5 plumbing: 2 ranks x 2 KV heads each, all-gather reassembles
    the query heads in KV-head order on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, heads, rows, group, gathered in out:
        assert heads != "error", rows
        assert heads == ([0, 1] if r == 0 else [2, 3]) and rows == list(range(6)) and group == [0, 1]
        for row in gathered:
            assert row == [float(i) for i in range(28)]


def test_head_shard_layout():
    assert fdist.head_shard_layout(8, 4) == (4, 2)   # Qwen2.5-7B on 8 GPUs: 4-way heads x 2 replicas
    assert fdist.head_shard_layout(8, 8) == (8, 1)
    assert fdist.head_shard_layout(1, 4) == (1, 1)
    heads, rows, group = fdist.head_shard_of(5, 8, 4, 16)
    assert list(heads) == [1] and rows == range(8, 16) and group == [4, 5, 6, 7]
