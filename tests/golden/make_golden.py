"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package ``tierkv`` read-only from
/root/reference/pkg/src and records its outputs on seeded, bf16-representable
inputs.  The fixtures travel with the repo; nothing at test time reads
/root/reference.  Every case names the reference function it exercises.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from tierkv.attention import (AttentionState, dense_decode,  # noqa: E402
                              sparse_decode, sparsity_error)
from tierkv.blocktable import BlockTable, PhysicalPool  # noqa: E402
from tierkv.config import Config, HeadId  # noqa: E402
from tierkv.scoring import (MinMaxMeta, build_minmax, rerank_due,  # noqa: E402
                            score_pages, select_topk, update_minmax)
from tierkv.tiering import promoted_delta  # noqa: E402
from tierkv.trace import gen_synthetic_kv  # noqa: E402

from oracle.flexicache_oracle import bf16_round  # noqa: E402


def minmax_cases(out):
    """scoring.py:72-90 build_minmax and :59-69 update_minmax."""
    rng = np.random.default_rng(101)
    for name, (t, d, ps) in {"a": (70, 16, 16), "b": (257, 128, 16),
                             "c": (5, 8, 4), "d": (1, 128, 16)}.items():
        keys = bf16_round(rng.standard_normal((t, d)) * rng.uniform(0.5, 4))
        meta = build_minmax(keys, ps)
        n = meta.n_pages
        out[f"minmax_{name}_keys"] = keys
        out[f"minmax_{name}_ps"] = np.int64(ps)
        out[f"minmax_{name}_mins"] = meta.mins[:n].copy()
        out[f"minmax_{name}_maxs"] = meta.maxs[:n].copy()
        out[f"minmax_{name}_fill"] = meta.fill[:n].copy()
        # incremental path must agree with the vectorised one
        inc = MinMaxMeta(d, ps)
        for i in range(t):
            if i % ps == 0:
                inc.add_page()
            update_minmax(inc, i // ps, keys[i])
        assert np.array_equal(inc.mins[:n], meta.mins[:n])


def score_cases(out):
    """scoring.py:102-111 score_pages; GQA group sum over G query heads."""
    rng = np.random.default_rng(202)
    for name, (n_pages, d, ps, g) in {"a": (64, 128, 16, 4), "b": (300, 128, 16, 7),
                                      "c": (17, 64, 16, 1)}.items():
        keys = bf16_round(rng.standard_normal((n_pages * ps - 3, d)))
        meta = build_minmax(keys, ps)
        qs = bf16_round(rng.standard_normal((g, d)))
        per_q = np.stack([score_pages(qs[j], meta) for j in range(g)])
        out[f"score_{name}_keys"] = keys
        out[f"score_{name}_ps"] = np.int64(ps)
        out[f"score_{name}_qs"] = qs
        out[f"score_{name}_per_q"] = per_q
        total = np.zeros(meta.n_pages)
        for j in range(g):
            total = total + per_q[j]
        out[f"score_{name}_group"] = total


def select_cases(js):
    """scoring.py:164-193 select_topk: known answers + tie-heavy random cases."""
    cases = [
        ([0.1, 5.0, 3.0, 4.0], 2, []),          # test_scoring.py:137-139
        ([9.0, 8.0, 7.0, 0.0], 2, [3]),         # :142-146
        ([1.0, 2.0, 2.0, 2.0], 2, []),          # :149-151
        ([1.0, 2.0], 8, []),                    # :154-156
        ([5.0, 1.0, 9.0, 9.0], 2, []),
        ([5.0, 1.0, 9.0, 9.0], 1, []),
        ([0.0, -0.0, 0.0, -1.0], 2, []),        # signed zero ties
        ([-3.0, -1.0, -2.0, -1.0, -5.0], 3, [4]),
    ]
    rng = np.random.default_rng(303)
    for _ in range(200):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 140))
        scores = rng.integers(-4, 5, size=n).astype(float) * 0.5
        pinned = [n - 1] if rng.random() < 0.8 else []
        cases.append((scores.tolist(), k, pinned))
    for _ in range(40):
        n = int(rng.integers(100, 2100))
        scores = bf16_round(rng.standard_normal(n) * 10).tolist()
        cases.append((scores, 128, [n - 1]))
    js["select"] = [dict(scores=s, k=k, pinned=p,
                         pages=list(select_topk(np.array(s), k, pinned=tuple(p)).pages))
                    for s, k, p in cases]


def attention_cases(out):
    """attention.py:76-111 dense/sparse decode on bf16-representable inputs."""
    rng = np.random.default_rng(404)
    specs = {"a": (70, 128, 16, [0, 2, 4]), "b": (64, 128, 16, [0, 1, 2, 3]),
             "c": (1, 128, 16, [0]), "d": (500, 64, 16, [1, 5, 9, 31]),
             "e": (2048 + 7, 128, 16, list(range(0, 129, 3)))}
    for name, (t, d, ps, pages) in specs.items():
        keys = bf16_round(rng.standard_normal((1, 1, t, d)))
        vals = bf16_round(rng.standard_normal((1, 1, t, d)))
        q = bf16_round(rng.standard_normal(d))
        st = AttentionState(keys, vals, page_size_tokens=ps)
        out[f"attn_{name}_keys"] = keys[0, 0]
        out[f"attn_{name}_vals"] = vals[0, 0]
        out[f"attn_{name}_q"] = q
        out[f"attn_{name}_ps"] = np.int64(ps)
        out[f"attn_{name}_pages"] = np.array(pages, dtype=np.int64)
        out[f"attn_{name}_sparse"] = sparse_decode(q, st, HeadId(0, 0), pages)
        out[f"attn_{name}_dense"] = dense_decode(q, st, HeadId(0, 0))
    # composed chain: summaries -> score -> select(pin last) -> dense vs sparse
    keys = bf16_round(rng.standard_normal((1, 2, 400, 64)))
    vals = bf16_round(rng.standard_normal((1, 2, 400, 64)))
    st = AttentionState(keys, vals, page_size_tokens=16)
    queries = bf16_round(rng.standard_normal((6, 1, 2, 64)))
    stats = sparsity_error(st, queries, budget=8)
    out["sperr_keys"], out["sperr_vals"], out["sperr_queries"] = keys, vals, queries
    out["sperr_errors"] = stats.errors


def recycle_cases(js):
    """blocktable.py:296-357 recycle, known answers and a random differential."""
    res = []
    rng = np.random.default_rng(505)
    specs = [((0, 1, 2, 3), (0, 1, 6, 7), 8), ((0, 1, 2, 3), (0, 1, 2), 8),
             ((0, 1, 2, 3), (0, 1, 2, 3, 6), 8), ((0, 1, 2, 3), (4, 5, 6, 7), 8)]
    for _ in range(60):
        n = int(rng.integers(4, 40))
        k1 = int(rng.integers(1, n + 1))
        k2 = int(rng.integers(1, n + 1))
        specs.append((tuple(np.sort(rng.choice(n, k1, replace=False)).tolist()),
                      tuple(np.sort(rng.choice(n, k2, replace=False)).tolist()), n))
    h = HeadId(0, 0)
    for old, new, n in specs:
        pool = PhysicalPool(128)
        t = BlockTable(pool, 1, 1, requests_cap=1, pages_cap=4)
        t.add_request("r")
        for _ in range(n):
            t.allocate_page("r", h)
        drop = [p for p in range(n) if p not in old]
        if drop:
            t.evict_many("r", h, drop)
        row_before = t._table[0, 0, 0, :n].tolist()
        free_before = list(pool._free)
        plan = t.recycle("r", h, old, new, slow_resident=range(n))
        res.append(dict(old=list(old), new=list(new), n=n, row_before=row_before,
                        free_before=free_before,
                        row_after=t._table[0, 0, 0, :n].tolist(),
                        free_after=list(pool._free),
                        evicted=list(plan.evicted), promoted=list(plan.promoted),
                        reassigned=[list(x) for x in plan.reassigned],
                        freed=list(plan.freed_blocks),
                        fresh=[list(x) for x in plan.fresh_allocs],
                        copies=[list(x) for x in plan.copies]))
    js["recycle"] = res
    js["promoted_delta"] = [dict(old=[0, 1, 2], new=[1, 2, 5, 7],
                                 out=list(promoted_delta((0, 1, 2), (1, 2, 5, 7)))),
                            dict(old=[], new=[3], out=list(promoted_delta((), (3,)))),
                            dict(old=[3], new=[3], out=list(promoted_delta((3,), (3,))))]
    # allocate_page_all_heads order: table[row, :, :, n] = allocate_many(L*H)
    pool = PhysicalPool(200)
    t = BlockTable(pool, 3, 4, requests_cap=2, pages_cap=2)
    t.add_request("a")
    t.add_request("b")
    for _ in range(3):
        t.allocate_page_all_heads("a")
        t.allocate_page_all_heads("b")
    js["alloc_all_heads"] = dict(L=3, H=4, table_a=t._table[t._rows["a"], :, :, :3].tolist(),
                                 table_b=t._table[t._rows["b"], :, :, :3].tolist(),
                                 free_top=pool._free[-5:])


def schedule_cases(js):
    """scoring.py:196-202 rerank_due."""
    class P:
        def is_unstable(self, h):
            return h == HeadId(0, 0)
    js["rerank_due"] = dict(
        stable=[s for s in range(1, 49) if rerank_due(HeadId(0, 1), s, P(), 16)],
        unstable=[s for s in range(1, 49) if rerank_due(HeadId(0, 0), s, P(), 16)])


def kv_gen_cases(out):
    """trace.py:217-225 gen_synthetic_kv draw order."""
    cfg = Config(num_layers=2, kv_heads_per_layer=3, head_dim=8)
    k, v = gen_synthetic_kv(cfg, 5)
    out["gen_kv_k"], out["gen_kv_v"] = k, v


def main():
    out: dict = {}
    js: dict = {}
    minmax_cases(out)
    score_cases(out)
    attention_cases(out)
    kv_gen_cases(out)
    select_cases(js)
    recycle_cases(js)
    schedule_cases(js)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **out)
    with open(os.path.join(HERE, "golden_cases.json"), "w") as fh:
        json.dump(js, fh)
    print("wrote", len(out), "arrays and", sum(len(v) if isinstance(v, list) else 1
                                                for v in js.values()), "cases")


if __name__ == "__main__":
    main()
