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
