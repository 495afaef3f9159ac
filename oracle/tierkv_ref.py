"""The UNMODIFIED reference ``tierkv`` timed on the host cores (BENCH
INFRASTRUCTURE ONLY: used by ``bench.py --impl reference`` and its
``cpu_baseline``; never imported by the product).

``tierkv`` is pure Python/numpy, so it is installed once into the git-ignored
``baseline/_ref`` (``pip install --no-index --no-build-isolation --no-deps
--target baseline/_ref <copy of /root/reference/pkg>``) and
travels to the GPU box with the repo snapshot.  One head unit of a decode
step runs the reference's own calls, composed for GQA exactly as the oracle
(SURVEY.md §8 a3/a6):

* ``update_minmax`` (scoring.py:59-69) of the appended key into its page;
* when the head is due (``rerank_due``, scoring.py:196-202): ``score_pages``
  (scoring.py:102-111) for each of the G query heads, summed in ascending g,
  then ``select_topk`` (scoring.py:164-193) with the last page pinned;
* ``sparse_decode`` (attention.py:85-111) for each of the G query heads over
  the head's selection.

Units are independent and fan out over a fork pool of host
processes with one BLAS thread each.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(HERE, "baseline", "_ref")

_W: dict = {}


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "tierkv"))


def _import():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import tierkv  # noqa: F401  (the installed reference, not a copy in this repo)
    from tierkv import attention, scoring
    from tierkv.config import HeadId
    return attention, scoring, HeadId


def _bf16(x):
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000))
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def setup(ctx: int, heads: int, d: int, g: int, k: int, seed: int = 12345) -> None:
    attention, scoring, HeadId = _import()
    rng = np.random.default_rng(seed)
    keys = _bf16(rng.standard_normal((1, heads, ctx, d)))
    vals = _bf16(rng.standard_normal((1, heads, ctx, d)))
    state = attention.AttentionState(keys=keys, values=vals, page_size_tokens=16)
    _W.update(state=state, g=g, k=k, heads=heads, d=d,
              metas=[state.minmax_for(HeadId(0, h)) for h in range(heads)],
              q=_bf16(rng.standard_normal((heads, g, d))),
              knew=_bf16(rng.standard_normal((heads, d))))
    _W["sel"] = [_select(h) for h in range(heads)]


def _select(h):
    _, scoring, _ = _import()
    meta = _W["metas"][h]
    qs = _W["q"][h]
    scores = scoring.score_pages(qs[0], meta)
    for gg in range(1, qs.shape[0]):
        scores = scores + scoring.score_pages(qs[gg], meta)
    return scoring.select_topk(scores, _W["k"], pinned=(meta.n_pages - 1,))


def limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def unit(job):
    """One (KV head, decode step): (head index, due) -> output checksum."""
    attention, scoring, HeadId = _import()
    h, due = job
    # the appended key opens a page (32k context: every page is full)
    scratch = scoring.MinMaxMeta(_W["d"], 16)
    page = scratch.add_page()
    scoring.update_minmax(scratch, page, _W["knew"][h])
    sel = _select(h) if due else _W["sel"][h]
    state, qs = _W["state"], _W["q"][h]
    acc = 0.0
    for gg in range(qs.shape[0]):
        acc += float(attention.sparse_decode(qs[gg], state, HeadId(0, h), sel)[0])
    return acc


def run_steps(*, ctx, heads, d, g, k, due_frac, units_per_step, steps, warmup, cores, seed=12345):
    """Wall seconds for ``steps`` samples of ``units_per_step`` head units
    (after ``warmup``), on ``cores`` fork-pool processes."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    limit_blas()
    setup(ctx, heads, d, g, k, seed)
    n_due = int(round(due_frac * units_per_step))
    jobs = [(i % heads, i < n_due) for i in range(units_per_step)]
    import multiprocessing as mp
    with mp.get_context("fork").Pool(cores, initializer=limit_blas) as pool:
        for _ in range(max(1, warmup)):
            pool.map(unit, jobs, chunksize=1)
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(unit, jobs, chunksize=1)
        return time.perf_counter() - t0
