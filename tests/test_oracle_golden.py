"""Pin the CPU oracle to the reference: every golden fixture produced by the
reference (tests/golden/make_golden.py) must be reproduced by oracle/.

CPU only; bit-exact wherever the reference arithmetic is reproduced in the
same order (min/max, select, recycle), 1e-12 relative where numpy reduction
order may differ (score sums, float64 attention)."""

import numpy as np
import pytest

from oracle import flexicache_oracle as O


@pytest.mark.parametrize("name", ["a", "b", "c", "d"])
def test_minmax_build_matches_reference(golden_arrays, name):
    g = golden_arrays
    keys, ps = g[f"minmax_{name}_keys"], int(g[f"minmax_{name}_ps"])
    mins, maxs, fill = O.minmax_build(keys, ps)
    assert np.array_equal(mins, g[f"minmax_{name}_mins"])
    assert np.array_equal(maxs, g[f"minmax_{name}_maxs"])
    assert np.array_equal(fill, g[f"minmax_{name}_fill"])


@pytest.mark.parametrize("name", ["a", "b", "c", "d"])
def test_minmax_incremental_matches_reference(golden_arrays, name):
    g = golden_arrays
    keys, ps = g[f"minmax_{name}_keys"], int(g[f"minmax_{name}_ps"])
    n = O.pages_for_tokens(keys.shape[0], ps)
    mins = np.full((n, keys.shape[1]), np.inf)
    maxs = np.full((n, keys.shape[1]), -np.inf)
    fill = np.zeros(n, dtype=np.int32)
    for t in range(keys.shape[0]):
        O.minmax_update(mins, maxs, fill, t // ps, keys[t], ps)
    assert np.array_equal(mins, g[f"minmax_{name}_mins"])
    assert np.array_equal(maxs, g[f"minmax_{name}_maxs"])


def test_minmax_update_rejections():
    mins, maxs = np.zeros((1, 4)), np.zeros((1, 4))
    fill = np.zeros(1, dtype=np.int32)
    with pytest.raises(ValueError):
        O.minmax_update(mins, maxs, fill, 0, np.zeros(5), 2)
    with pytest.raises(ValueError):
        O.minmax_update(mins, maxs, fill, 1, np.zeros(4), 2)
    O.minmax_update(mins, maxs, fill, 0, np.zeros(4), 2)
    O.minmax_update(mins, maxs, fill, 0, np.zeros(4), 2)
    with pytest.raises(ValueError, match="full"):
        O.minmax_update(mins, maxs, fill, 0, np.zeros(4), 2)


@pytest.mark.parametrize("name", ["a", "b", "c"])
def test_scores_match_reference(golden_arrays, name):
    g = golden_arrays
    keys, ps, qs = g[f"score_{name}_keys"], int(g[f"score_{name}_ps"]), g[f"score_{name}_qs"]
    mins, maxs, _ = O.minmax_build(keys, ps)
    for j in range(qs.shape[0]):
        np.testing.assert_allclose(O.score_pages(qs[j], mins, maxs),
                                   g[f"score_{name}_per_q"][j], rtol=1e-12, atol=0)
    np.testing.assert_allclose(O.group_scores(qs, mins, maxs), g[f"score_{name}_group"],
                               rtol=1e-12, atol=1e-12)


def test_select_matches_reference(golden_cases):
    for case in golden_cases["select"]:
        got = O.select_topk(np.array(case["scores"]), case["k"], case["pinned"])
        assert list(got) == case["pages"], case
        fast = O.select_topk_fast(np.array(case["scores"]), case["k"], case["pinned"])
        assert list(fast) == case["pages"]


def test_select_rejections():
    with pytest.raises(ValueError):
        O.select_topk(np.array([1.0]), 1, pinned=(5,))
    with pytest.raises(ValueError):
        O.select_topk(np.array([1.0, 2.0]), 1, pinned=(0, 1))
    with pytest.raises(ValueError):
        O.select_topk(np.array([1.0]), 0)


@pytest.mark.parametrize("name", ["a", "b", "c", "d", "e"])
def test_attention_matches_reference(golden_arrays, name):
    g = golden_arrays
    keys, vals, q = g[f"attn_{name}_keys"], g[f"attn_{name}_vals"], g[f"attn_{name}_q"]
    ps, pages = int(g[f"attn_{name}_ps"]), g[f"attn_{name}_pages"]
    np.testing.assert_allclose(O.sparse_decode(q, keys, vals, ps, pages),
                               g[f"attn_{name}_sparse"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(O.dense_decode(q, keys, vals), g[f"attn_{name}_dense"],
                               rtol=1e-12, atol=1e-14)


def test_sparse_full_budget_is_dense_bitwise(golden_arrays):
    g = golden_arrays
    keys, vals, q = g["attn_a_keys"], g["attn_a_vals"], g["attn_a_q"]
    n = O.pages_for_tokens(keys.shape[0], 16)
    assert np.array_equal(O.sparse_decode(q, keys, vals, 16, range(n)),
                          O.dense_decode(q, keys, vals))


def test_residency_guard():
    rng = np.random.default_rng(6)
    k, v = rng.standard_normal((64, 8)), rng.standard_normal((64, 8))
    with pytest.raises(O.OracleConsistencyError, match="residency"):
        O.sparse_decode(rng.standard_normal(8), k, v, 16, (0, 1, 2), resident=(0, 2))


def test_composed_sparsity_error_matches_reference(golden_arrays):
    """attention.py:128-160: summaries -> score -> select(pin last) -> attend."""
    g = golden_arrays
    keys, vals, queries = g["sperr_keys"], g["sperr_vals"], g["sperr_queries"]
    errs = []
    T = keys.shape[2]
    last = O.pages_for_tokens(T, 16) - 1
    for s in range(queries.shape[0]):
        for h in range(keys.shape[1]):
            mins, maxs, _ = O.minmax_build(keys[0, h], 16)
            q = queries[s, 0, h]
            sel = O.select_topk(O.score_pages(q, mins, maxs), 8, pinned=(last,))
            ref = O.dense_decode(q, keys[0, h], vals[0, h])
            out = O.sparse_decode(q, keys[0, h], vals[0, h], 16, sel)
            errs.append(np.linalg.norm(out - ref) / np.linalg.norm(ref))
    np.testing.assert_allclose(errs, g["sperr_errors"], rtol=1e-9, atol=1e-15)


def test_recycle_matches_reference(golden_cases):
    for c in golden_cases["recycle"]:
        row = np.array(c["row_before"], dtype=np.int32)
        pool = O.Pool(128)
        pool.free = list(c["free_before"])
        pool.is_free[:] = False
        pool.is_free[pool.free] = True
        plan = O.recycle(row, pool, c["old"], c["new"], slow_resident=range(c["n"]))
        assert row.tolist() == c["row_after"]
        assert pool.free == c["free_after"]
        assert list(plan["evicted"]) == c["evicted"]
        assert list(plan["promoted"]) == c["promoted"]
        assert [list(x) for x in plan["reassigned"]] == c["reassigned"]
        assert list(plan["freed_blocks"]) == c["freed"]
        assert [list(x) for x in plan["fresh_allocs"]] == c["fresh"]
        assert [list(x) for x in plan["copies"]] == c["copies"]


def test_promoted_delta_matches_reference(golden_cases):
    for c in golden_cases["promoted_delta"]:
        assert list(O.promoted_delta(c["old"], c["new"])) == c["out"]


def test_alloc_all_heads_order(golden_cases):
    """blocktable.py:248-263: table[row,:,:,n] = allocate_many(L*H) reshaped."""
    c = golden_cases["alloc_all_heads"]
    L, H = c["L"], c["H"]
    pool = O.Pool(200)
    ta = np.zeros((L, H, 3), dtype=np.int32)
    tb = np.zeros((L, H, 3), dtype=np.int32)
    for n in range(3):
        ta[:, :, n] = pool.allocate_many(L * H).reshape(L, H)
        tb[:, :, n] = pool.allocate_many(L * H).reshape(L, H)
    assert ta.tolist() == c["table_a"] and tb.tolist() == c["table_b"]
    assert pool.free[-5:] == c["free_top"]


def test_rerank_schedule_matches_reference(golden_cases):
    c = golden_cases["rerank_due"]
    assert [s for s in range(1, 49) if O.rerank_due(False, s, 16)] == c["stable"]
    assert [s for s in range(1, 49) if O.rerank_due(True, s, 16)] == c["unstable"]


def test_gen_synthetic_kv_draw_order(golden_arrays):
    k, v = O.gen_synthetic_kv(2, 3, 5, 8, seed=12345)
    assert np.array_equal(k, golden_arrays["gen_kv_k"])
    assert np.array_equal(v, golden_arrays["gen_kv_v"])


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(10000) * 100
    want = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(O.bf16_round(x), want)
