"""End-to-end parity of the batched decode step (DecodeEngine) against the
oracle, step by step: append -> summaries (bit-exact) -> due-head scoring
and selection (exact given the GPU scores; oracle-equal outside the tie band)
-> GQA sparse attention over sel ∪ appended pages (bf16 2e-2 / fp32 1e-5)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import flexicache_oracle as O  # noqa: E402

PS = 16


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _round(x, dtype):
    return O.bf16_round(x) if dtype == torch.bfloat16 else O.f32_round(x)


def run_engine_vs_oracle(*, B, L, H, G, D, T0, steps, K, R, frac, dtype, seed, use_graph,
                         ragged=False, tiering=False, run_kernel=None, fused=False, spread=0):
    from paper_2511_00868_b200.config import HeadId
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    rng = np.random.default_rng(seed)
    prof = HeadProfile.first_n(L, H, frac)
    if spread:  # the first `spread` KV heads of every layer unstable (mixed layers)
        prof = HeadProfile(model_id="spread", n_layers=L, n_heads_per_layer=H, fraction=spread / H,
                           unstable=tuple(HeadId(l, h) for l in range(L) for h in range(spread)))
    unstable = prof.mask()
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D,
                       ctx_cap_tokens=T0 + steps + 64, topk_pages=K, rerank_period=R,
                       profile=prof, dtype=dtype, tiering=tiering)
    eng.run_kernel = run_kernel
    eng.fused_score_attend = fused
    dev = eng.device
    lens = [T0 + (17 * b if ragged else 0) for b in range(B)]
    keys = {}
    vals = {}
    for b in range(B):
        k = _round(rng.standard_normal((L, H, lens[b], D)), dtype)
        v = _round(rng.standard_normal((L, H, lens[b], D)), dtype)
        for l in range(L):
            for h in range(H):
                keys[b, l, h] = k[l, h]
                vals[b, l, h] = v[l, h]
        eng.prefill(b, torch.as_tensor(k).to(dev, dtype), torch.as_tensor(v).to(dev, dtype))
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    worst = 0.0
    tie_mismatch = 0
    for step in range(steps):
        t = eng.t
        q = _round(rng.standard_normal((L, B, H * G, D)), dtype)
        kn = _round(rng.standard_normal((L, B, H, D)), dtype)
        vn = _round(rng.standard_normal((L, B, H, D)), dtype)
        eng.q.copy_(torch.as_tensor(q))
        eng.k_new.copy_(torch.as_tensor(kn))
        eng.v_new.copy_(torch.as_tensor(vn))
        first = not eng.selected
        eng.step(use_graph=use_graph)
        eng.store.check_errors()
        sel = eng.store.sel.cpu().numpy()
        n_sel = eng.store.n_sel.cpu().numpy()
        out = eng.out.double().cpu().numpy()
        summ = eng.store.summaries.double().cpu().numpy()
        table = eng.store.table.cpu().numpy()
        for b in range(B):
            for l in range(L):
                for h in range(H):
                    keys[b, l, h] = np.vstack([keys[b, l, h], kn[l, b, h][None]])
                    vals[b, l, h] = np.vstack([vals[b, l, h], vn[l, b, h][None]])
                    kk, vv = keys[b, l, h], vals[b, l, h]
                    n_tok = kk.shape[0]
                    n_pages = O.pages_for_tokens(n_tok, PS)
                    mins, maxs, _ = O.minmax_build(kk, PS)
                    # (1) summaries bit-exact
                    assert np.array_equal(summ[b, l, h, :n_pages, 0], mins)
                    assert np.array_equal(summ[b, l, h, :n_pages, 1], maxs)
                    due = first or unstable[l, h] or t % R == 0
                    # the selection row also holds the page the next token opens
                    # (fc_step_advance appends it); this step attended pages < n_pages
                    gsel = tuple(p for p in sel[b, l, h, :n_sel[b, l, h]].tolist() if p < n_pages)
                    qs = q[l, b, h * G:(h + 1) * G]
                    if due:
                        # (2) selection: oracle select on oracle scores, tie band
                        osc = O.group_scores(qs, mins, maxs)
                        osel = O.select_topk_fast(osc, K, (n_pages - 1,))
                        if gsel != osel:
                            kth = np.sort(osc[:-1])[::-1][min(K, n_pages) - 2] if n_pages > K else 0.0
                            band = 1e-4 * (np.abs(qs).sum(axis=0) @ np.maximum(np.abs(mins), np.abs(maxs)).T).max()
                            for p in set(gsel) ^ set(osel):
                                assert abs(osc[p] - kth) <= band, (b, l, h, p)
                            tie_mismatch += 1
                    if tiering and not unstable[l, h]:
                        # stable heads keep exactly their selection in HBM
                        # (boundary residency check, simulator.py:526-531)
                        n_alloc = O.pages_for_tokens(n_tok + 1, PS)
                        resident = tuple(np.flatnonzero(table[b, l, h, :n_alloc]).tolist())
                        assert resident == tuple(sel[b, l, h, :n_sel[b, l, h]].tolist()), (step, b, l, h)
                    # (3) attention over the GPU's attended set
                    pages = O.attended_pages(gsel, n_pages)
                    want = O.gqa_sparse_decode(qs, kk, vv, PS, pages)
                    got = out[l, b, h * G:(h + 1) * G]
                    err = np.linalg.norm(got - want) / np.linalg.norm(want)
                    worst = max(worst, err)
                    assert err <= tol, (step, b, l, h, err)
    return worst, tie_mismatch, eng


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_engine_matches_oracle(dtype):
    worst, ties, eng = run_engine_vs_oracle(B=2, L=2, H=2, G=4, D=128, T0=300, steps=12, K=8,
                                            R=4, frac=0.5, dtype=dtype, seed=5, use_graph=False)
    assert ties <= 2


def test_engine_graph_replay_matches_oracle():
    worst, ties, eng = run_engine_vs_oracle(B=3, L=2, H=2, G=4, D=128, T0=250, steps=20, K=6,
                                            R=4, frac=0.5, dtype=torch.bfloat16, seed=6,
                                            use_graph=True, ragged=True)
    assert len(eng._graphs) == 2  # rerank and plain step graphs both replayed


def test_engine_qwen_group7_d128():
    run_engine_vs_oracle(B=1, L=2, H=2, G=7, D=128, T0=200, steps=6, K=5, R=2, frac=0.5,
                         dtype=torch.bfloat16, seed=7, use_graph=True)


def test_engine_d64_small_context_dense_budget():
    """n_pages <= K: every page selected (budget covers the pool)."""
    run_engine_vs_oracle(B=2, L=1, H=2, G=2, D=64, T0=40, steps=30, K=16, R=8, frac=0.5,
                         dtype=torch.bfloat16, seed=8, use_graph=True)


def test_page_table_injective_and_conserving():
    worst, ties, eng = run_engine_vs_oracle(B=2, L=2, H=2, G=4, D=128, T0=100, steps=40, K=4,
                                            R=4, frac=0.5, dtype=torch.bfloat16, seed=9,
                                            use_graph=True)
    st = eng.store
    table = st.table.cpu().numpy()
    live = table[table != 0]
    assert np.unique(live).size == live.size            # check_injective (blocktable.py:389-392)
    assert st.free_count() + live.size + 1 == st.n_blocks  # check_conservation (:394-400)


def test_engine_tiered_rerank_fetch_matches_oracle():
    """Two-tier mode: stable heads hold only their selection in HBM; reranks
    recycle blocks and fetch promoted pages from pinned host memory; pages
    filled during decode are offloaded once.  Attention after every fetch
    must still equal the oracle (fetched K/V are the written K/V)."""
    worst, ties, eng = run_engine_vs_oracle(B=2, L=2, H=4, G=4, D=128, T0=400, steps=24, K=6,
                                            R=4, frac=0.5, dtype=torch.bfloat16, seed=10,
                                            use_graph=True, tiering=True)
    assert int(eng.fetched_pages.item()) > 0
    eng.store.check_errors()


@pytest.fixture
def head_aligned_scoring():
    """Force the head-aligned scoring kernel (one CTA per head) that the
    launcher otherwise picks only when the batch has >= SMs/2 heads."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    lib = _lib.load()
    lib.fc_debug_score_mode.argtypes = [ctypes.c_int]
    lib.fc_debug_score_mode(1)
    yield
    lib.fc_debug_score_mode(-1)


@pytest.mark.parametrize("dtype,D,G", [(torch.bfloat16, 128, 4), (torch.float32, 128, 4),
                                       (torch.bfloat16, 64, 2), (torch.float32, 64, 7)])
def test_engine_head_aligned_scoring_matches_oracle(head_aligned_scoring, dtype, D, G):
    # T0 = 1500 tokens -> ~94 candidate pages: two 64-page chunks, the last partial
    worst, ties, eng = run_engine_vs_oracle(B=2, L=2, H=2, G=G, D=D, T0=1500, steps=10, K=8,
                                            R=4, frac=0.5, dtype=dtype, seed=11, use_graph=True,
                                            ragged=True)
    assert ties <= 2


@pytest.mark.parametrize("dtype,D,G", [(torch.bfloat16, 128, 4), (torch.float32, 128, 4),
                                       (torch.bfloat16, 64, 7), (torch.float32, 64, 2)])
def test_engine_fused_score_attend_matches_oracle(head_aligned_scoring, dtype, D, G):
    """fc_score_attend: each head's CTA scores, selects and attends."""
    worst, ties, eng = run_engine_vs_oracle(B=2, L=2, H=2, G=G, D=D, T0=1500, steps=10, K=8,
                                            R=4, frac=0.5, dtype=dtype, seed=18, use_graph=True,
                                            ragged=True, fused=True)
    assert eng.launches_per_step(1) == 3  # fused layer 0, attention layer 1, advance
    assert ties <= 2


@pytest.mark.parametrize("D,G,spread", [(128, 4, 1), (128, 7, 2), (64, 4, 3)])
def test_engine_balanced_scoring_matches_oracle(head_aligned_scoring, D, G, spread):
    """fc_score_attend_balanced (plain steps of layers with some heads due):
    the due heads' pages scored in equal shares by every CTA of a one-wave
    grid, then each head's CTA selects (when due) and attends."""
    worst, ties, eng = run_engine_vs_oracle(B=3, L=2, H=4, G=G, D=D, T0=1500, steps=10, K=8,
                                            R=4, frac=0.5, dtype=torch.bfloat16, seed=23, use_graph=True,
                                            ragged=True, fused=True, spread=spread)
    assert eng._use_balanced(0, "plain", False) and not eng._use_balanced(0, "rerank", False)
    assert ties <= 2


def test_engine_balanced_scoring_tiered(head_aligned_scoring):
    run_engine_vs_oracle(B=2, L=2, H=4, G=4, D=128, T0=700, steps=16, K=6, R=4, frac=0.5,
                         dtype=torch.bfloat16, seed=24, use_graph=True, tiering=True, fused=True, spread=2)


def test_balanced_bitwise_equals_two_launch():
    """At config 2's batch (16 rows x 8 KV heads, 2 due per layer) the
    balanced fused launch gives the same scores, selections, summaries and
    outputs, bit for bit, as the balanced scoring kernel followed by
    fc_sparse_decode (same per-page score arithmetic, same attention)."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    from paper_2511_00868_b200.config import HeadId
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    B, L, H, G, D, T, K, R = 16, 2, 8, 4, 128, 6000, 32, 16
    prof = HeadProfile(model_id="spread", n_layers=L, n_heads_per_layer=H, fraction=0.25,
                       unstable=tuple(HeadId(l, h) for l in range(L) for h in range(2)))
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                       topk_pages=K, rerank_period=R, profile=prof)
    assert eng.store.score_attend_balanced_supported(B) >= B * H
    for b in range(B):
        for l in range(L):
            eng.prefill_layer(b, l, device_normal((H, T - 37 * b, D), seed=3 * b + l),
                              device_normal((H, T - 37 * b, D), seed=100 + 3 * b + l), alloc=(l == 0))
    eng.q.copy_(device_normal(tuple(eng.q.shape), seed=5))
    eng.step()  # initial selection of every head
    st = eng.store
    eng.q.copy_(device_normal(tuple(eng.q.shape), seed=6))
    eng.k_new.copy_(device_normal(tuple(eng.k_new.shape), seed=7))
    eng.v_new.copy_(device_normal(tuple(eng.v_new.shape), seed=8))
    snap = [t.clone() for t in (st.sel, st.n_sel, st.summaries, st.kv_pool)]
    lib = _lib.load()
    lib.fc_debug_score_mode.argtypes = [ctypes.c_int]
    lib.fc_debug_score_mode(0)  # the balanced scoring kernel
    try:
        for l in range(L):
            st.score_select(l, eng.q[l], eng.unstable, R, K, B, extra_tokens=1, kv_prefetch=l > 0)
            st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=eng.att_bound, extra_tokens=1,
                             attend_appended=False, k_new=eng.k_new[l], v_new=eng.v_new[l])
    finally:
        lib.fc_debug_score_mode(-1)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (st.sel, st.n_sel, st.summaries, eng.out, st.scores)]
    for t, v in zip((st.sel, st.n_sel, st.summaries, st.kv_pool), snap):
        t.copy_(v)
    for l in range(L):
        st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                 kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])
    torch.cuda.synchronize()
    st.check_errors()
    for got, want in zip((st.sel, st.n_sel, st.summaries, eng.out, st.scores), ref):
        assert torch.equal(got, want)
    assert int(st.score_counters.abs().sum()) == 0  # left zero for the next launch
    # chunked attention of the scored heads (their pages cut into chunks that
    # the owner and any CTA with no work left claim; the last to finish a head
    # merges): the same selections and summaries; the outputs differ only by
    # the order of the softmax merge
    for t, v in zip((st.sel, st.n_sel, st.summaries, st.kv_pool), snap):
        t.copy_(v)
    st.balanced_helpers = True
    try:
        for it in range(3):  # repeatedly: the launch epoch keeps earlier launches' words stale
            for t, v in zip((st.sel, st.n_sel, st.summaries, st.kv_pool), snap):
                t.copy_(v)
            for l in range(L):
                st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                         kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])
            torch.cuda.synchronize()
            st.check_errors()
            for got, want in zip((st.sel, st.n_sel, st.summaries, st.scores), (ref[0], ref[1], ref[2], ref[4])):
                assert torch.equal(got, want)
            err = (eng.out.float() - ref[3].float()).norm() / ref[3].float().norm()
            assert float(err) < 5e-3, float(err)
            glob = st._bal_ws[4 * B * H * 4:(4 * B * H + 2) * 4].view(torch.int32).tolist()
            assert glob == [(it + 1) * L, 0]  # one epoch per launch, exit count back to zero
    finally:
        st.balanced_helpers = False


def test_engine_fused_tiered(head_aligned_scoring):
    run_engine_vs_oracle(B=2, L=2, H=4, G=4, D=128, T0=400, steps=16, K=6, R=4, frac=0.5,
                         dtype=torch.bfloat16, seed=19, use_graph=True, tiering=True, fused=True)


@pytest.mark.parametrize("dtype,D,G", [(torch.bfloat16, 128, 4), (torch.float32, 128, 4),
                                       (torch.bfloat16, 64, 7), (torch.float32, 64, 2)])
def test_engine_fused_clusters_match_oracle(dtype, D, G):
    """fc_score_attend at small batches: each head is scored, selected and
    attended by a cluster of CTAs (keys gathered in rank 0 through DSMEM,
    rank 0 selects, every rank attends its share, DSMEM merge)."""
    worst, ties, eng = run_engine_vs_oracle(B=3, L=2, H=2, G=G, D=D, T0=1500, steps=10, K=8,
                                            R=4, frac=0.5, dtype=dtype, seed=20, use_graph=True,
                                            ragged=True, fused=True)
    assert eng.store.score_attend_supported(eng.B) > 1  # a cluster per head
    assert ties <= 2


def test_engine_fused_clusters_tiered():
    run_engine_vs_oracle(B=2, L=2, H=4, G=4, D=128, T0=700, steps=16, K=6, R=4, frac=0.5,
                         dtype=torch.bfloat16, seed=21, use_graph=True, tiering=True, fused=True)


def test_engine_head_aligned_tiered(head_aligned_scoring):
    run_engine_vs_oracle(B=2, L=2, H=4, G=4, D=128, T0=400, steps=16, K=6, R=4, frac=0.5,
                         dtype=torch.bfloat16, seed=12, use_graph=True, tiering=True)


def test_early_heads_bitwise_equal_to_serialized():
    """Attention of heads the scoring launch does not select starts without
    waiting for it (PDL); the outputs, selections and summaries must be
    bit-identical to the fully serialized schedule."""
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    B, L, H, G, D, T, K, R = 4, 4, 4, 4, 128, 3000, 16, 4
    outs = []
    for early in (False, True):
        eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                           topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25))
        eng.early_heads = early
        eng.run_kernel = False  # early heads belong to the per-layer kernel
        for b in range(B):
            for l in range(L):
                eng.prefill_layer(b, l, device_normal((H, T + 7 * b, D), seed=4 * b + l),
                                  device_normal((H, T + 7 * b, D), seed=100 + 4 * b + l), alloc=(l == 0))
        gen = torch.Generator(device="cuda")
        gen.manual_seed(21)
        rec = []
        for step in range(10):
            eng.q.normal_(generator=gen)
            eng.k_new.normal_(generator=gen)
            eng.v_new.normal_(generator=gen)
            eng.step()
            rec.append(eng.out.clone())
        torch.cuda.synchronize()
        eng.store.check_errors()
        outs.append((torch.stack(rec), eng.store.sel.clone(), eng.store.summaries.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.fixture
def balanced_attention():
    """Force the balanced all-SM attention variant (not auto-selected: the
    cluster-per-head kernel measured faster) so it stays covered."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    lib = _lib.load()
    lib.fc_debug_attn_mode.argtypes = [ctypes.c_int]
    lib.fc_debug_attn_mode(1)
    yield
    lib.fc_debug_attn_mode(0)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_engine_balanced_attention_matches_oracle(balanced_attention, dtype):
    worst, ties, eng = run_engine_vs_oracle(B=3, L=2, H=2, G=4, D=128, T0=700, steps=12, K=8,
                                            R=4, frac=0.5, dtype=dtype, seed=13, use_graph=True,
                                            ragged=True, run_kernel=False)
    assert ties <= 2


def test_engine_balanced_attention_tiered(balanced_attention):
    run_engine_vs_oracle(B=2, L=2, H=4, G=7, D=128, T0=400, steps=16, K=6, R=4, frac=0.5,
                         dtype=torch.bfloat16, seed=14, use_graph=True, tiering=True)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_engine_per_layer_attention_matches_oracle(dtype):
    """The per-layer cluster kernel (fc_sparse_decode, the default) over
    several unscored layers in a row (KV staged while the previous layer
    drains)."""
    run_engine_vs_oracle(B=2, L=4, H=2, G=4, D=128, T0=500, steps=10, K=8, R=4, frac=0.25,
                         dtype=dtype, seed=15, use_graph=True, ragged=True)


@pytest.mark.parametrize("dtype,D,G", [(torch.bfloat16, 128, 4), (torch.float32, 128, 4),
                                       (torch.bfloat16, 64, 7), (torch.float32, 64, 2)])
def test_engine_layer_runs_match_oracle(dtype, D, G):
    """fc_sparse_decode_layers over runs of several layers (1/8 of the heads
    unstable: layer 0 scored every step, layers 1-5 one persistent launch
    between reranks); ragged rows, graph replay, rerank steps."""
    worst, ties, eng = run_engine_vs_oracle(B=3, L=6, H=2, G=G, D=D, T0=600, steps=12, K=8, R=4,
                                            frac=0.125, dtype=dtype, seed=16, use_graph=True,
                                            ragged=True, run_kernel=True)
    assert eng.launches_per_step(1) == 3  # score(0), run [0, 6), advance
    assert ties <= 2


def test_engine_layer_runs_tiered():
    run_engine_vs_oracle(B=2, L=4, H=4, G=4, D=128, T0=400, steps=16, K=6, R=4, frac=0.25,
                         dtype=torch.bfloat16, seed=17, use_graph=True, tiering=True, run_kernel=True)
