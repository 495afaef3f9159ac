"""CPU baseline timing of the hot path with the oracle (TEST/BENCH
INFRASTRUCTURE ONLY: used by bench.py's ``cpu_baseline`` leg and
``--impl reference``; never by the product).

The reference is pure Python/numpy and cannot travel to the
GPU box, so the baseline runs the oracle restatement of the same algorithm
(``kind: "port"``): per KV head and decode step, the reference chain
  group score_pages (scoring.py:102-111, summed over G)  +  select_topk
  (scoring.py:164-193, last page pinned)  when the head is due, and
  sparse_decode (attention.py:85-111) for each of its G query heads over the
  selected pages, plus update_minmax (scoring.py:59-69) for the new key.
Work is split into independent head units and fanned out
over a fork pool of host cores (``OPENBLAS_NUM_THREADS=1``).
A decode step of config 2 has B*L*H head units of which a fraction
u + (1-u)/R are due for scoring (unstable every step, stable every R).
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import flexicache_oracle as O

_W: dict = {}  # worker globals (fork inherits)


def _setup(ctx: int, heads: int, d: int, g: int, k: int, seed: int) -> None:
    rng = np.random.default_rng(seed)
    T = ctx
    _W["keys"] = [O.bf16_round(rng.standard_normal((T, d))) for _ in range(heads)]
    _W["vals"] = [O.bf16_round(rng.standard_normal((T, d))) for _ in range(heads)]
    _W["meta"] = [O.minmax_build(kk, 16) for kk in _W["keys"]]
    _W["q"] = O.bf16_round(rng.standard_normal((heads, g, d)))
    _W["k"] = k
    _W["sel"] = [O.select_topk_fast(O.group_scores(_W["q"][h], m[0], m[1]), k,
                                    (O.pages_for_tokens(T, 16) - 1,))
                 for h, m in enumerate(_W["meta"])]


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def _unit(job):
    """One head for one decode step: (head index, due) -> output checksum."""
    h, due = job
    keys, vals = _W["keys"][h], _W["vals"][h]
    mins, maxs, fill = _W["meta"][h]
    n_pages = mins.shape[0]
    qs = _W["q"][h]
    # update_minmax of the appended key on a scratch copy of the last page
    mn, mx, fl = mins[-1:].copy(), maxs[-1:].copy(), np.zeros(1, dtype=np.int32)
    O.minmax_update(mn, mx, fl, 0, keys[-1], 16)
    if due:
        sel = O.select_topk_fast(O.group_scores(qs, mins, maxs), _W["k"], (n_pages - 1,))
    else:
        sel = _W["sel"][h]
    out = O.gqa_sparse_decode(qs, keys, vals, 16, sel)
    return float(out[0, 0])


def time_units(*, ctx=32768, heads=8, d=128, g=4, k=128, due_frac=0.296875, n_units=64,
               cores=1, seed=12345, repeats=1):
    """Seconds per head unit (wall, with ``cores`` processes) for a unit mix
    whose due fraction matches the config.  Returns (sec_per_unit, n_units)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _limit_blas()
    _setup(ctx, heads, d, g, k, seed)
    n_due = int(round(due_frac * n_units))
    jobs = [(i % heads, i < n_due) for i in range(n_units)]
    _unit(jobs[0])  # warm caches / BLAS init
    if cores <= 1:
        t0 = time.perf_counter()
        for _ in range(repeats):
            for j in jobs:
                _unit(j)
        dt = time.perf_counter() - t0
    else:
        import multiprocessing as mp
        ctxm = mp.get_context("fork")
        with ctxm.Pool(cores, initializer=_limit_blas) as pool:
            pool.map(_unit, jobs[:cores])  # spin up
            t0 = time.perf_counter()
            for _ in range(repeats):
                pool.map(_unit, jobs, chunksize=max(1, n_units // (cores * 4)))
            dt = time.perf_counter() - t0
    return dt / (n_units * repeats), n_units * repeats


def tokens_per_s(sec_per_unit: float, *, batch: int, layers: int, heads: int) -> float:
    """Decode tokens/s of the whole config: one step = B*L*H head units."""
    step_s = sec_per_unit * batch * layers * heads
    return batch / step_s


def due_fraction(u: float, period: int) -> float:
    return u + (1.0 - u) / period


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


if __name__ == "__main__":
    spu, n = time_units(n_units=16, cores=1)
    print(f"1 core: {spu * 1e3:.2f} ms/unit -> {tokens_per_s(spu, batch=16, layers=32, heads=8):.3f} tok/s")
    c = host_cores()
    spu, n = time_units(n_units=8 * c, cores=c)
    print(f"{c} cores: {spu * 1e3:.2f} ms/unit -> {tokens_per_s(spu, batch=16, layers=32, heads=8):.3f} tok/s")
    _ = math
