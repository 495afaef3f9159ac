"""The persistent multi-layer attention kernel (fc_sparse_decode_layers) at
the config-2 head count (16 rows x 8 KV heads = 128 heads per layer), where
every head is cut across several warps and merged by the last arriver:

* outputs == float64 oracle on the GPU's own selection (bf16 2e-2) for
  sampled heads of every layer of the run, against the K/V read back from
  the pool;
* selections and summaries bit-identical to the per-layer kernel's engine
  (attention does not feed back into them);
* outputs deterministic (bit-identical across two engines);
* direct C-ABI call with an LSE output equals the per-layer fc_sparse_decode
  LSE within fp32 rounding.
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


@pytest.fixture(params=[0, 1], ids=["per_head_clusters", "warp_balanced"])
def run_mode(request):
    """fc_sparse_decode_layers kernel: 0 the per-head cluster persistent
    kernel (default where it fits), 1 the warp-balanced one."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    lib = _lib.load()
    lib.fc_debug_run_mode.argtypes = [ctypes.c_int]
    lib.fc_debug_run_mode(request.param)
    yield request.param
    lib.fc_debug_run_mode(0)


def _engine(run_kernel, B=16, L=4, H=8, G=4, D=128, T=2000, K=24, R=4, frac=0.25, steps=6, seed=3,
            fused=False):
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64 + 16 * B,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, frac))
    eng.run_kernel = run_kernel
    eng.fused_score_attend = fused
    for b in range(B):
        for l in range(L):
            n = T + 13 * b  # ragged rows
            eng.prefill_layer(b, l, device_normal((H, n, D), seed=100 * b + 2 * l),
                              device_normal((H, n, D), seed=100 * b + 2 * l + 1), alloc=(l == 0))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    outs = []
    for _ in range(steps):
        eng.q.normal_(generator=gen)
        eng.k_new.normal_(generator=gen)
        eng.v_new.normal_(generator=gen)
        eng.step()
        outs.append(eng.out.clone())
    torch.cuda.synchronize()
    eng.store.check_errors()
    return eng, torch.stack(outs)


def test_run_kernel_config2_heads_vs_oracle_and_per_layer(run_mode):
    eng_r, out_r = _engine(True)
    eng_p, out_p = _engine(False)
    st = eng_r.store
    assert torch.equal(st.sel, eng_p.store.sel)
    assert torch.equal(st.n_sel, eng_p.store.n_sel)
    assert torch.equal(st.summaries, eng_p.store.summaries)
    rel = (out_r.float() - out_p.float()).norm() / out_p.float().norm()
    assert rel < 1e-2, rel
    # oracle on sampled heads of every layer, last step
    B, L, H, G = eng_r.B, eng_r.L, eng_r.H, eng_r.G
    seq = st.seq_len.cpu().numpy()
    sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
    out = eng_r.out.double().cpu().numpy()
    q = eng_r.q.double().cpu().numpy()
    for (b, h) in ((0, 0), (5, 3), (11, 7), (15, 4)):
        for l in range(L):
            n_tok = int(seq[b])
            n_pages = -(-n_tok // PS)
            k, v = st.gather(b, l, h, n_pages)
            k = k[:n_tok].double().cpu().numpy()
            v = v[:n_tok].double().cpu().numpy()
            pages = [p for p in sel[b, l, h, :n_sel[b, l, h]].tolist() if p < n_pages]
            want = O.gqa_sparse_decode(q[l, b, h * G:(h + 1) * G], k, v, PS, pages)
            got = out[l, b, h * G:(h + 1) * G]
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2, (b, l, h)


def test_run_kernel_deterministic(run_mode):
    _, a = _engine(True, B=8, L=3, steps=4, seed=9)
    _, b = _engine(True, B=8, L=3, steps=4, seed=9)
    assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_layers_call_lse_matches_per_layer(dtype, run_mode):
    """Direct calls (no fused append, attend_appended): the run kernel over
    layers [0, L) vs fc_sparse_decode per layer, outputs and LSE."""
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    B, L, H, G, D, T, K = 12, 3, 4, 4, 128, 1500, 16
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 200,
                       topk_pages=K, rerank_period=4, profile=HeadProfile.first_n(L, H, 1.0), dtype=dtype)
    for b in range(B):
        for l in range(L):
            eng.prefill_layer(b, l, device_normal((H, T + 9 * b, D), seed=b * 7 + l).to(dtype),
                              device_normal((H, T + 9 * b, D), seed=1000 + b * 7 + l).to(dtype), alloc=(l == 0))
    eng.q.normal_()
    eng.step()  # initial selection of every head
    st = eng.store
    q = torch.randn_like(eng.q)
    o_run = torch.zeros_like(eng.out)
    o_ref = torch.zeros_like(eng.out)
    lse_run = torch.zeros((L, B * H * G), dtype=torch.float32, device=q.device)
    lse_ref = torch.zeros_like(lse_run)
    mp = eng.att_bound
    st.sparse_decode_layers(0, L, q, o_run, B, max_pages=mp, lse=lse_run, extra_tokens=1, attend_appended=False)
    for l in range(L):
        st.sparse_decode(l, q[l], o_ref[l], B, max_pages=mp, lse=lse_ref[l], extra_tokens=1,
                         attend_appended=False)
    torch.cuda.synchronize()
    st.check_errors()
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    assert ((o_run.float() - o_ref.float()).norm() / o_ref.float().norm()).item() < tol
    assert torch.allclose(lse_run, lse_ref, rtol=1e-5, atol=1e-5)


def test_fused_score_attend_config2_heads_vs_oracle():
    """fc_score_attend (one CTA per head scores, selects and attends) as the
    engine's path for scored layers at 128 heads: selection == select_topk
    over the GPU's own scores (exact), attention == float64 oracle on that
    selection, summaries bit-identical to the unfused engine's."""
    eng_f, out_f = _engine(False, L=2, frac=0.5, steps=5, seed=21, fused=True)
    assert eng_f.fused_score_attend and eng_f.store.score_attend_supported(eng_f.B)
    assert eng_f.launches_per_step(1) == 1 + 1 + 1  # fused layer 0, attention layer 1, advance
    st = eng_f.store
    B, L, H, G = eng_f.B, eng_f.L, eng_f.H, eng_f.G
    seq = st.seq_len.cpu().numpy()
    sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
    scores = st.scores.cpu().numpy()
    out = eng_f.out.double().cpu().numpy()
    q = eng_f.q.double().cpu().numpy()
    K = eng_f.K
    for bh in (0, 37, 90, 127):  # layer 0 (unstable, scored every step, scored last)
        b, h = divmod(bh, H)
        n_tok = int(seq[b])
        n_pages = -(-n_tok // PS)
        row = scores[bh, :n_pages - 1].astype(np.float64)
        want_sel = O.select_topk_fast(np.append(row, 0.0), K, (n_pages - 1,))
        got_sel = tuple(x for x in sel[b, 0, h, :n_sel[b, 0, h]].tolist() if x < n_pages)
        assert got_sel == want_sel
        k, v = st.gather(b, 0, h, n_pages)
        k = k[:n_tok].double().cpu().numpy()
        v = v[:n_tok].double().cpu().numpy()
        want = O.gqa_sparse_decode(q[0, b, h * G:(h + 1) * G], k, v, PS, list(got_sel))
        got = out[0, b, h * G:(h + 1) * G]
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2, bh


def test_fused_and_unfused_summaries_identical():
    eng_f, _ = _engine(False, B=16, L=2, frac=0.5, steps=4, seed=22, fused=True)
    eng_u, _ = _engine(False, B=16, L=2, frac=0.5, steps=4, seed=22, fused=False)
    assert torch.equal(eng_f.store.summaries, eng_u.store.summaries)
    assert torch.equal(eng_f.store.table, eng_u.store.table)


@pytest.mark.parametrize("B", [1, 4])
def test_run_kernel_small_batch_clusters_vs_oracle(B, run_mode):
    """Small batches: the per-head persistent kernel splits each head over a
    cluster of up to 16 CTAs (DSMEM merge) for every layer of the run."""
    eng, out = _engine(True, B=B, L=4, H=8, T=3000, K=32, frac=0.125, steps=5, seed=30 + B)
    st = eng.store
    L, H, G = eng.L, eng.H, eng.G
    seq = st.seq_len.cpu().numpy()
    sel, n_sel = st.sel.cpu().numpy(), st.n_sel.cpu().numpy()
    o = eng.out.double().cpu().numpy()
    q = eng.q.double().cpu().numpy()
    for b in range(B):
        for (l, h) in ((0, 0), (1, 3), (2, 5), (3, 7)):
            n_tok = int(seq[b])
            n_pages = -(-n_tok // PS)
            k, v = st.gather(b, l, h, n_pages)
            k = k[:n_tok].double().cpu().numpy()
            v = v[:n_tok].double().cpu().numpy()
            pages = [p for p in sel[b, l, h, :n_sel[b, l, h]].tolist() if p < n_pages]
            want = O.gqa_sparse_decode(q[l, b, h * G:(h + 1) * G], k, v, PS, pages)
            got = o[l, b, h * G:(h + 1) * G]
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2, (b, l, h)


def test_fused_one_cta_bitwise_equal_to_two_launches():
    """fc_score_attend with one CTA per head (head-aligned mode) computes the
    same page keys as the head-aligned scoring kernel and attends with the
    same warp decomposition as fc_sparse_decode: selections, outputs and LSE
    bit-identical to the two launches."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    lib = _lib.load()
    lib.fc_debug_score_mode.argtypes = [ctypes.c_int]
    lib.fc_debug_score_mode(1)  # head-aligned: one CTA per head in both paths
    try:
        B, L, H, G, D, T, K = 4, 1, 4, 4, 128, 3000, 16
        eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                           topk_pages=K, rerank_period=4, profile=HeadProfile.first_n(L, H, 1.0))
        for b in range(B):
            eng.prefill_layer(b, 0, device_normal((H, T + 11 * b, D), seed=b),
                              device_normal((H, T + 11 * b, D), seed=50 + b), alloc=True)
        st = eng.store
        q = device_normal(tuple(eng.q[0].shape), seed=7)
        res = []
        for fused in (False, True):
            out = torch.zeros_like(eng.out[0])
            lse = torch.zeros(B * H * G, dtype=torch.float32, device=q.device)
            if fused:
                st.score_attend(0, q, eng.unstable, 4, K, out, B, force_due=True, extra_tokens=1, lse=lse)
            else:
                st.score_select(0, q, eng.unstable, 4, K, B, force_due=True, extra_tokens=1)
                st.sparse_decode(0, q, out, B, max_pages=eng.att_bound, lse=lse, extra_tokens=1,
                                 attend_appended=False, n_ctas=1)  # one CTA per head, as fused
            torch.cuda.synchronize()
            st.check_errors()
            res.append((st.sel.clone(), st.n_sel.clone(), out, lse))
        for x, y in zip(*res):
            assert torch.equal(x, y)
    finally:
        lib.fc_debug_score_mode(-1)


@pytest.mark.parametrize("force_due", [False, True])
def test_fused_mixed_clusters_match_uniform(force_due):
    """fc_score_attend_map (mixed clusters: scored heads split over a cluster,
    the others one CTA each, idle padding CTAs) against the uniform one-CTA
    launch: selections identical, outputs of heads attended alone
    bit-identical, split heads within bf16 rounding, LSE within fp32
    rounding.  force_due: every head is scored, so heads attended alone also
    score and select alone."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    from paper_2511_00868_b200.synthetic import device_normal
    lib = _lib.load()
    lib.fc_debug_score_mode.argtypes = [ctypes.c_int]
    B, L, H, G, D, T, K = 2, 1, 8, 4, 128, 6000, 32
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                       topk_pages=K, rerank_period=4, profile=HeadProfile.first_n(L, H, 0.25))
    for b in range(B):
        eng.prefill_layer(b, 0, device_normal((H, T + 11 * b, D), seed=b),
                          device_normal((H, T + 11 * b, D), seed=50 + b), alloc=True)
    st = eng.store
    st.step.fill_(1)  # a plain step: only the unstable heads are due unless forced
    unstable = [h for h in range(H) if eng.unstable.view(L, H)[0, h].item()]
    assert len(unstable) == 2
    q = device_normal(tuple(eng.q[0].shape), seed=7)

    def run(cta_map=None, cluster=0):
        out = torch.zeros_like(eng.out[0])
        lse = torch.zeros(B * H * G, dtype=torch.float32, device=q.device)
        st.sel.zero_()
        st.n_sel.zero_()
        st.score_attend(0, q, eng.unstable, 4, K, out, B, force_due=force_due, extra_tokens=1, lse=lse,
                        cta_map=cta_map, cluster=cluster)
        torch.cuda.synchronize()
        st.check_errors()
        return st.sel.clone(), st.n_sel.clone(), out, lse

    lib.fc_debug_score_mode(1)  # uniform reference: one CTA per head
    try:
        ref = run()
    finally:
        lib.fc_debug_score_mode(-1)
    S = 4
    split, alone = [], []
    for b in range(B):
        for h in range(H):
            (split if h in unstable else alone).append(b * H + h)
    m = [bh for bh in split for _ in range(S)] + [bh | (1 << 30) for bh in alone]
    m += [-1] * (-len(m) % S) + [-1] * S  # padding and one idle cluster
    assert st.score_attend_map_fits(len(m), S)
    got = run(torch.tensor(m, dtype=torch.int32, device="cuda"), S)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
    o_ref, o_got = ref[2].view(B, H, G, D), got[2].view(B, H, G, D)
    for bh in alone:
        assert torch.equal(o_got[bh // H, bh % H], o_ref[bh // H, bh % H]), bh
    for bh in split:
        a, r = o_got[bh // H, bh % H].float(), o_ref[bh // H, bh % H].float()
        assert ((a - r).norm() / r.norm()).item() < 1e-2, bh
    assert torch.allclose(got[3], ref[3], rtol=1e-5, atol=1e-5)


def test_mixed_cluster_map_plan():
    """The engine's plan for a small batch at long context: every head
    appears once, scored heads split over whole clusters, the grid fits."""
    from paper_2511_00868_b200.store import KVStore
    st = KVStore(batch_cap=8, layers=1, kv_heads=8, group=4, head_dim=128, pages_cap=8200, n_blocks=64,
                 sel_cap=140, dtype=torch.bfloat16, device="cuda")
    plan = st.mixed_cluster_map(8, [0, 1], 8192, 128)
    assert plan is not None
    m, S = plan
    m = m.cpu().tolist()
    assert len(m) % S == 0 and st.score_attend_map_fits(len(m), S)
    heads = [e & ~(1 << 30) for e in m if e >= 0]
    split = [e for e in m if e >= 0 and not e & (1 << 30)]
    assert sorted(set(heads)) == list(range(64))
    assert sorted(set(split)) == sorted(b * 8 + h for b in range(8) for h in (0, 1))
    assert all(split.count(e) == S for e in set(split))
    # config 2's shape (16 rows, 2 kv heads of 8 scored): no mixed grid fits one wave
    st2 = KVStore(batch_cap=16, layers=1, kv_heads=8, group=4, head_dim=128, pages_cap=2100, n_blocks=64,
                  sel_cap=140, dtype=torch.bfloat16, device="cuda")
    assert st2.mixed_cluster_map(16, [0, 1], 2048, 128) is None
