"""Parity at the BASELINE configurations (BASELINE.json:configs), every head
against the float64 oracle:

* config 1 exactly — one Llama-3.1-8B-shaped layer (32 q / 8 KV heads,
  d = 128), 8k context, page 16, top-K 128 pages, batch 1, 50 % stable heads,
  R = 8, 24 decode steps (initial selection + reranks at t = 8, 16, 24):
  summaries bit-exact, selections equal to ``select_topk`` on the GPU's own
  scores exactly and to the oracle's float64 selection outside the fp32 tie
  band (band hits counted and bounded), attention within 2e-2 (bf16 store) /
  1e-5 (fp32 store) of float64 on the GPU's selection; also two-tier;
* one config-2-shape layer — 32k context, 16 requests × 8 KV heads, K = 128:
  every head's selection against the float64 oracle under the tie band, every
  head's attention, summaries bit-exact (keys read back from the pool);
* the -inf merge guard of ``attn_kernel``: more cluster CTAs than attended
  pages (explicit ``n_ctas``, and the auto split of a ragged batch).

Reference chain: ``sparsity_error`` (attention.py:128-160) — summaries ->
score -> select(pin last) -> sparse attention; ``select_topk``
(scoring.py:164-193); ``rerank_due`` (scoring.py:196-202).

Tie band (documented): the GPU scores in fp32 from the same
summaries with w = [Σ_g q_g⁻ | Σ_g q_g⁺]; a length-n fp32 dot product is
within n·u·Σ|terms| (u = 2⁻²⁴) of the exact value, so two pages can swap
order only when their float64 scores differ by less than
    band = 2·(2d + G + 2)·2⁻²⁴·max_p Σ_i Σ_g |q_gi|·max(|min_pi|, |max_pi|).
"""

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


def tie_band(qs, mins, maxs):
    D, G = mins.shape[1], qs.shape[0]
    mag = np.abs(qs).sum(axis=0) @ np.maximum(np.abs(mins), np.abs(maxs)).T
    return 2.0 * (2 * D + G + 2) * 2.0 ** -24 * float(mag.max())


def check_selection(gsel, qs, mins, maxs, K, stats):
    """GPU selection vs the oracle's float64 select_topk(pin last): equal, or
    every differing page within the tie band of the K-th score."""
    n_pages = mins.shape[0]
    osc = O.group_scores(qs, mins, maxs)
    osel = O.select_topk_fast(osc, K, (n_pages - 1,))
    stats["heads"] += 1
    if gsel == osel:
        return
    assert len(gsel) == len(osel)
    band = tie_band(qs, mins, maxs)
    kth = np.sort(osc[:-1])[::-1][min(K, n_pages) - 2]
    for p in set(gsel) ^ set(osel):
        assert abs(osc[p] - kth) <= band, (p, osc[p], kth, band)
    stats["band_heads"] += 1
    stats["band_pages"] += len(set(gsel) ^ set(osel)) // 2


def _new_stats():
    return {"heads": 0, "band_heads": 0, "band_pages": 0}


# ---------------------------------------------------------------------------
# config 1

@pytest.mark.parametrize("dtype,tiering", [(torch.bfloat16, False), (torch.float32, False),
                                           (torch.bfloat16, True)])
def test_config1_every_head_vs_oracle(dtype, tiering):
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    B, L, H, G, D, T0, K, R, STEPS = 1, 1, 8, 4, 128, 8192, 128, 8, 24
    prof = HeadProfile.first_n(L, H, 0.5)           # 50 % stable (config 1)
    unstable = prof.mask()
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T0 + STEPS + 64,
                       topk_pages=K, rerank_period=R, profile=prof, dtype=dtype, tiering=tiering)
    dev = eng.device
    # gen_synthetic_kv draw order (trace.py:217-225), seed cfg.rng_seed = 12345
    rng = np.random.default_rng(12345)
    k0 = _round(rng.standard_normal((L, H, T0, D)), dtype)
    v0 = _round(rng.standard_normal((L, H, T0, D)), dtype)
    eng.prefill(0, torch.as_tensor(k0).to(dev, dtype), torch.as_tensor(v0).to(dev, dtype))
    keys = [k0[0, h] for h in range(H)]
    vals = [v0[0, h] for h in range(H)]
    qrng = np.random.default_rng(12346)             # queries: seed + 1 (cli.py:325)
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    stats, worst, reranks = _new_stats(), 0.0, 0
    for step in range(STEPS):
        t = eng.t
        first = not eng.selected
        reranks += int(t % R == 0)
        q = _round(qrng.standard_normal((L, B, H * G, D)), dtype)
        kn = _round(qrng.standard_normal((L, B, H, D)), dtype)
        vn = _round(qrng.standard_normal((L, B, H, D)), dtype)
        eng.q.copy_(torch.as_tensor(q))
        eng.k_new.copy_(torch.as_tensor(kn))
        eng.v_new.copy_(torch.as_tensor(vn))
        eng.step(use_graph=step > 1)
        eng.store.check_errors()
        st = eng.store
        sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
        out = eng.out.double().cpu().numpy()
        summ = st.summaries.double().cpu().numpy()
        scores = st.scores.double().cpu().numpy()
        table = st.table.cpu().numpy()
        for h in range(H):
            keys[h] = np.vstack([keys[h], kn[0, 0, h][None]])
            vals[h] = np.vstack([vals[h], vn[0, 0, h][None]])
            n_tok = keys[h].shape[0]
            n_pages = O.pages_for_tokens(n_tok, PS)
            mins, maxs, _ = O.minmax_build(keys[h], PS)
            assert np.array_equal(summ[0, 0, h, :n_pages, 0], mins), (step, h)
            assert np.array_equal(summ[0, 0, h, :n_pages, 1], maxs), (step, h)
            gsel = tuple(p for p in sel[0, 0, h, :n_sel[0, 0, h]].tolist() if p < n_pages)
            qs = q[0, 0, h * G:(h + 1) * G]
            if first or unstable[0, h] or t % R == 0:
                assert len(gsel) == K
                # exact: select_topk on the GPU's own fp32 scores (pinned last page)
                own = O.select_topk_fast(np.append(scores[h, :n_pages - 1], 0.0), K, (n_pages - 1,))
                assert gsel == own, (step, h)
                check_selection(gsel, qs, mins, maxs, K, stats)
            if tiering and not unstable[0, h]:
                n_alloc = O.pages_for_tokens(n_tok + 1, PS)
                resident = tuple(np.flatnonzero(table[0, 0, h, :n_alloc]).tolist())
                assert resident == tuple(sel[0, 0, h, :n_sel[0, 0, h]].tolist()), (step, h)
            want = O.gqa_sparse_decode(qs, keys[h], vals[h], PS, O.attended_pages(gsel, n_pages))
            got = out[0, 0, h * G:(h + 1) * G]
            assert np.all(np.isfinite(got))
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            worst = max(worst, err)
            assert err <= tol, (step, h, err)
    assert reranks >= 3
    if tiering:
        # write-once ledger over every full page, the ones filled during decode
        # included (tiering.py:99-157; decode-time offloads are device-recorded)
        full = (T0 + STEPS) // PS
        for h in range(H):
            got = eng.tier.slow_pages(0, (0, h))
            assert got == (set() if unstable[0, h] else set(range(full))), h
    # 8 heads at the initial step + 4 unstable per plain step + 8 per rerank
    assert stats["heads"] == 8 + 4 * (STEPS - 1 - reranks) + 8 * reranks
    # band hits are rare (fp32 vs float64 near-ties); report them
    print(f"config1 {dtype} tiering={tiering}: worst rel err {worst:.2e}, "
          f"{stats['band_heads']}/{stats['heads']} head selections differ inside the tie band "
          f"({stats['band_pages']} page swaps)")
    assert stats["band_heads"] <= max(2, stats["heads"] // 20)


# ---------------------------------------------------------------------------
# config-2 shape, one layer

@pytest.mark.parametrize("dtype,B,fused", [(torch.bfloat16, 16, True), (torch.bfloat16, 16, False),
                                           (torch.float32, 4, True)])
def test_config2_layer_every_head_vs_oracle(dtype, B, fused):
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    L, H, G, D, T, K, R = 1, 8, 4, 128, 32768, 128, 16
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25), dtype=dtype)
    eng.fused_score_attend = fused
    for b in range(B):
        eng.prefill_layer(b, 0, device_normal((H, T, D), seed=2 * b, dtype=dtype),
                          device_normal((H, T, D), seed=2 * b + 1, dtype=dtype), alloc=True)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    st = eng.store
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    stats, worst = _new_stats(), 0.0
    for step in range(2):           # initial selection (all due), then a plain step (2 unstable heads)
        t = eng.t
        first = not eng.selected
        eng.q.copy_(torch.randn(eng.q.shape, generator=gen, device="cuda").to(dtype))
        eng.k_new.copy_(torch.randn(eng.k_new.shape, generator=gen, device="cuda").to(dtype))
        eng.v_new.copy_(torch.randn(eng.v_new.shape, generator=gen, device="cuda").to(dtype))
        eng.step(use_graph=False)
        st.check_errors()
        sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
        seq = st.seq_len.cpu().numpy()
        out = eng.out.double().cpu().numpy()
        q = eng.q.double().cpu().numpy()
        summ = st.summaries[:, 0]
        for b in range(B):
            n_tok = int(seq[b])
            n_pages = O.pages_for_tokens(n_tok, PS)
            for h in range(H):
                k, v = st.gather(b, 0, h, n_pages)
                k = k[:n_tok].double().cpu().numpy()
                v = v[:n_tok].double().cpu().numpy()
                mins, maxs, _ = O.minmax_build(k, PS)
                s = summ[b, h, :n_pages].double().cpu().numpy()
                assert np.array_equal(s[:, 0], mins) and np.array_equal(s[:, 1], maxs), (b, h)
                gsel = tuple(p for p in sel[b, 0, h, :n_sel[b, 0, h]].tolist() if p < n_pages)
                qs = q[0, b, h * G:(h + 1) * G]
                if first or eng.profile.is_unstable((0, h)) or t % R == 0:
                    assert len(gsel) == K
                    check_selection(gsel, qs, mins, maxs, K, stats)
                want = O.gqa_sparse_decode(qs, k, v, PS, O.attended_pages(gsel, n_pages))
                got = out[0, b, h * G:(h + 1) * G]
                assert np.all(np.isfinite(got))
                err = np.linalg.norm(got - want) / np.linalg.norm(want)
                worst = max(worst, err)
                assert err <= tol, (step, b, h, err)
    assert stats["heads"] == B * H + B * 2
    print(f"config2 layer {dtype} B={B} fused={fused}: worst rel err {worst:.2e}, "
          f"{stats['band_heads']}/{stats['heads']} selections inside the tie band")
    assert stats["band_heads"] <= max(2, stats["heads"] // 20)


# ---------------------------------------------------------------------------
# the -inf guard of attn_kernel's merges (cluster ranks with no pages)

@pytest.mark.parametrize("n_ctas", [2, 4, 16])
def test_sparse_decode_more_ctas_than_pages(n_ctas):
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    B, L, H, G, D, T, K = 1, 1, 2, 4, 128, 20, 8
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=256,
                       topk_pages=K, rerank_period=4, profile=HeadProfile.first_n(L, H, 0.5))
    rng = np.random.default_rng(3)
    k0 = O.bf16_round(rng.standard_normal((L, H, T, D)))
    v0 = O.bf16_round(rng.standard_normal((L, H, T, D)))
    eng.prefill(0, torch.as_tensor(k0).cuda().bfloat16(), torch.as_tensor(v0).cuda().bfloat16())
    eng.step(use_graph=False)                 # initial selection: both pages
    st = eng.store
    q = torch.as_tensor(O.bf16_round(rng.standard_normal((B, H * G, D)))).cuda().bfloat16()
    out = torch.full_like(q, float("nan"))
    lse = torch.full((B * H * G,), float("nan"), dtype=torch.float32, device="cuda")
    st.sparse_decode(0, q, out, B, max_pages=eng.att_bound, n_ctas=n_ctas, lse=lse, extra_tokens=0,
                     attend_appended=True)
    torch.cuda.synchronize()
    st.check_errors()
    assert torch.isfinite(out).all() and torch.isfinite(lse).all()
    k, v = [], []
    n_tok = int(st.seq_len[0])
    for h in range(H):
        kk, vv = st.gather(0, 0, h, O.pages_for_tokens(n_tok, PS))
        k.append(kk[:n_tok].double().cpu().numpy())
        v.append(vv[:n_tok].double().cpu().numpy())
    qn = q.double().cpu().numpy()
    for h in range(H):
        want = O.gqa_sparse_decode(qn[0, h * G:(h + 1) * G], k[h], v[h], PS, range(O.pages_for_tokens(n_tok, PS)))
        got = out[0, h * G:(h + 1) * G].double().cpu().numpy()
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2


def test_ragged_batch_short_row_auto_split():
    """A 20-token row next to a 32k row, per-layer attention kernel (run
    kernel off): the auto cluster size is sized from the longest row, so the
    short row's heads have fewer pages than CTAs."""
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    B, L, H, G, D, K, R = 2, 1, 8, 4, 128, 128, 64
    lens = (20, 32768)
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=lens[1] + 64,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.0))
    eng.run_kernel = False
    for b in range(B):
        eng.prefill_layer(b, 0, device_normal((H, lens[b], D), seed=b),
                          device_normal((H, lens[b], D), seed=10 + b), alloc=True)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    st = eng.store
    for step in range(3):                     # initial selection, then plain attention-only steps
        eng.q.normal_(generator=gen)
        eng.k_new.normal_(generator=gen)
        eng.v_new.normal_(generator=gen)
        eng.step(use_graph=step > 0)
        st.check_errors()
        assert torch.isfinite(eng.out).all(), step
    sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
    seq = st.seq_len.cpu().numpy()
    out = eng.out.double().cpu().numpy()
    q = eng.q.double().cpu().numpy()
    for b in range(B):
        n_tok = int(seq[b])
        n_pages = O.pages_for_tokens(n_tok, PS)
        for h in range(H):
            k, v = st.gather(b, 0, h, n_pages)
            k, v = k[:n_tok].double().cpu().numpy(), v[:n_tok].double().cpu().numpy()
            gsel = [p for p in sel[b, 0, h, :n_sel[b, 0, h]].tolist() if p < n_pages]
            want = O.gqa_sparse_decode(q[0, b, h * G:(h + 1) * G], k, v, PS, O.attended_pages(gsel, n_pages))
            got = out[0, b, h * G:(h + 1) * G]
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2, (b, h)
