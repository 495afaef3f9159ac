"""The serving loop on the decode path: requests join and leave the rows of
a DecodeEngine mid-stream (prefill, per-row initial selection, decode in the
batch graph, release of every page), under a fast-tier budget.  Checks: every
request finishes, no device error, every block back in the pool, and the
attention of a request that joined mid-stream equals the float64 oracle."""

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


def _setup(B=3, L=2, H=2, G=4, D=128, K=8, R=4, cap=2000, tiering=False):
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=cap,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.5), tiering=tiering)
    return eng


def test_serving_loop_requests_finish_and_blocks_return():
    from paper_2511_00868_b200.serving import Request, ServingLoop
    eng = _setup()
    L, H, D = eng.L, eng.H, eng.D
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)

    def make_prompt(req):
        g = torch.Generator(device="cuda")
        g.manual_seed(1000 + req.id)
        k = torch.randn((L, H, req.prompt_tokens, D), generator=g, device="cuda").bfloat16()
        v = torch.randn((L, H, req.prompt_tokens, D), generator=g, device="cuda").bfloat16()
        return k, v

    def feed(e):
        e.q.normal_(generator=gen)
        e.k_new.normal_(generator=gen)
        e.v_new.normal_(generator=gen)

    # the first three arrive together (every row busy), the rest trickle in
    reqs = [Request(i, 0.0 if i < 3 else 0.0005 * i, 300 + 97 * i, 4 + 3 * (i % 3)) for i in range(7)]
    loop = ServingLoop(eng, reqs, make_prompt, feed)
    m = loop.run()
    assert m.finished == len(reqs) and m.queued_at_end == 0
    assert m.output_tokens == sum(r.output_tokens - 1 for r in reqs)
    assert m.peak_batch == eng.B
    assert m.tpot_mean_s > 0 and m.ttft_mean_s > 0 and m.throughput_tokens_per_s > 0
    torch.cuda.synchronize()
    eng.store.check_errors()
    assert eng.store.free_count() == eng.store.n_blocks - 1  # every block back in the pool
    assert bool((eng.store.table == 0).all())


@pytest.mark.parametrize("tiering,hold", [(False, 0), (True, 0), (True, 6)])
def test_request_joining_mid_stream_matches_oracle(tiering, hold):
    """Row 1 joins while row 0 is decoding; its first decode steps (initial
    selection with its own query, then the batch graph; two-tier: offload
    after prefill on a side stream, eviction once it finished, reranks
    fetching promoted pages) match the oracle.  hold > 0 keeps each row's
    eviction pending for that many steps, so reranks (t = 4, 8) run while a
    row still holds every page (fc_rerank_recycle_rows skips it)."""
    eng = _setup(B=2, K=6, tiering=tiering)
    if tiering:
        eng.evict_hold_steps = hold
    L, H, G, D = eng.L, eng.H, eng.G, eng.D
    rng = np.random.default_rng(3)
    eng.start_serving()
    prompts = {}
    for row, T in ((0, 500), (1, 420)):
        k = O.bf16_round(rng.standard_normal((L, H, T, D)))
        v = O.bf16_round(rng.standard_normal((L, H, T, D)))
        prompts[row] = [k, v]
    eng.admit(0, torch.as_tensor(prompts[0][0]).cuda().bfloat16(), torch.as_tensor(prompts[0][1]).cuda().bfloat16())
    for step in range(10):
        if step == 3:
            eng.admit(1, torch.as_tensor(prompts[1][0]).cuda().bfloat16(),
                      torch.as_tensor(prompts[1][1]).cuda().bfloat16())
        q = O.bf16_round(rng.standard_normal((L, 2, H * G, D)))
        kn = O.bf16_round(rng.standard_normal((L, 2, H, D)))
        vn = O.bf16_round(rng.standard_normal((L, 2, H, D)))
        eng.q.copy_(torch.as_tensor(q))
        eng.k_new.copy_(torch.as_tensor(kn))
        eng.v_new.copy_(torch.as_tensor(vn))
        eng.step()
        torch.cuda.synchronize()
        eng.store.check_errors()
        if tiering and hold:
            # admitted at t = 1 and t = 4: evicted from t = 7 and t = 10 on
            assert eng.eviction_pending(0) == (eng.t - 1 < 7)
            assert eng.eviction_pending(1) == (step >= 3 and eng.t - 1 < 10)
            if eng.t - 1 >= 7:  # row 0 evicted: stable heads keep only their selection
                res = (eng.store.table[0] != 0).sum(-1).cpu()
                ns = eng.store.n_sel[0].cpu()
                st_mask = ~eng.unstable.bool().cpu().view(eng.L, eng.H)
                assert bool((res[st_mask] <= ns[st_mask] + 1).all())  # + the next page
        sel, n_sel = eng.store.sel.cpu().numpy(), eng.store.n_sel.cpu().numpy()
        out = eng.out.double().cpu().numpy()
        for row in (0, 1):
            if row == 1 and step < 3:
                continue
            k, v = prompts[row]
            k = np.concatenate([k, kn[:, row, :, None, :]], axis=2)
            v = np.concatenate([v, vn[:, row, :, None, :]], axis=2)
            prompts[row] = [k, v]
            n_tok = k.shape[2]
            n_pages = O.pages_for_tokens(n_tok, PS)
            for l in range(L):
                for h in range(H):
                    pages = [p for p in sel[row, l, h, :n_sel[row, l, h]].tolist() if p < n_pages]
                    assert pages and pages[-1] == n_pages - 1
                    want = O.gqa_sparse_decode(q[l, row, h * G:(h + 1) * G], k[l, h], v[l, h], PS, pages)
                    got = out[l, row, h * G:(h + 1) * G]
                    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 2e-2, (step, row, l, h)
    eng.retire(0)
    eng.retire(1)
    torch.cuda.synchronize()
    assert eng.store.free_count() == eng.store.n_blocks - 1


def test_tiered_serving_admits_more_requests():
    """Two-tier serving: FlexiCache's commit (stable heads keep their
    selection) admits more requests into the same pool than the
    all-resident commit; requests finish, the pool and the slow-tier ledger
    are released, no device error."""
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.serving import Request, ServingLoop
    from paper_2511_00868_b200.stability import HeadProfile
    B, L, H, G, D, K, R = 4, 2, 4, 4, 128, 6, 4
    T = 1600
    per_req_dense = ((T + 20) // PS + 1) * L * H
    n_blocks = 2 * per_req_dense + 1          # all-resident: two requests at a time
    peaks = {}
    for tiering in (False, True):
        eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                           topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25),
                           n_blocks=n_blocks, tiering=tiering)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(9)

        def make_prompt(req):
            g = torch.Generator(device="cuda")
            g.manual_seed(77 + req.id)
            k = torch.randn((L, H, req.prompt_tokens, D), generator=g, device="cuda").bfloat16()
            v = torch.randn((L, H, req.prompt_tokens, D), generator=g, device="cuda").bfloat16()
            return k, v

        def feed(e):
            e.q.normal_(generator=gen)
            e.k_new.normal_(generator=gen)
            e.v_new.normal_(generator=gen)

        reqs = [Request(i, 0.0, T, 12 + 4 * i) for i in range(6)]
        m = ServingLoop(eng, reqs, make_prompt, feed).run()
        torch.cuda.synchronize()
        eng.store.check_errors()
        assert m.finished == len(reqs)
        assert eng.store.free_count() == eng.store.n_blocks - 1
        if tiering:
            assert eng.tier.slow_bytes_used == 0 and not eng.tier._counts
            assert int(eng.fetched_pages.item()) > 0
        peaks[tiering] = m.peak_batch
    assert peaks[False] == 2 and peaks[True] > 2
