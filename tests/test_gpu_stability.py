"""Head-stability profiling on the GPU: fc_trace_overlap
intersections -> reports and classifications bit-identical to the
reference's (golden fixtures) and to the oracle on larger generated traces;
fc_trace_capture records the engine's selections as FXTK traces."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import GOLDEN  # noqa: E402
from oracle import stability_oracle as S  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def _tr(name):
    from paper_2511_00868_b200.trace import load_trace
    return load_trace(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("name,window,stride", [("w8", 8, 8), ("w8s4", 8, 4), ("w5s3", 5, 3)])
def test_report_bit_exact_vs_reference(trace_golden, name, window, stride):
    from paper_2511_00868_b200.stability import compute_stability_report
    rep = compute_stability_report(_tr("trace_planted.fxtk"), window=window, stride=stride)
    r = trace_golden["planted"][name]
    assert list(rep.window_starts) == r["window_starts"]
    assert _hx(rep.ts) == r["ts"] and _hx(rep.offset_rco) == r["offset_rco"]
    assert rep.degenerate_pairs == r["degenerate_pairs"]
    assert rep.bottom_counts(0.25).reshape(-1).tolist() == r["bottom_counts_25"]


def test_report_text_and_degenerate_pools(trace_golden, tmp_path):
    from paper_2511_00868_b200.config import Config
    from paper_2511_00868_b200.stability import compute_stability_report
    cfg = Config(num_layers=2, kv_heads_per_layer=4, topk_pages=16, stability_window=8)
    rep = compute_stability_report(_tr("trace_planted.fxtk"), cfg)
    p = tmp_path / "rep.txt"
    rep.save_text(p)
    assert p.read_text() == trace_golden["planted"]["report_text_w8"].replace("trace=planted", "trace=trace_planted")
    g = compute_stability_report(_tr("trace_growth.fxtk"), window=8, stride=4)
    r = trace_golden["growth"]
    assert _hx(g.ts) == r["ts"] and _hx(g.offset_rco) == r["offset_rco"]
    assert g.degenerate_pairs == r["degenerate_pairs"] > 0


def test_classify_and_temporal_vs_reference(trace_golden, tmp_path):
    from paper_2511_00868_b200.config import HeadId
    from paper_2511_00868_b200.stability import classify_heads, compute_stability_report, temporal_stability
    from paper_2511_00868_b200.trace import TopKTrace
    tr = _tr("trace_planted.fxtk")
    tr.sample_id = "planted"
    rep = compute_stability_report(tr, window=8)
    for frac in (0.25, 0.5):
        prof = classify_heads([rep], frac, model_id="planted-model", task="qa")
        r = trace_golden["planted"][f"classify_{frac}"]
        assert [list(h) for h in prof.unstable] == r["unstable"]
        assert prof.bottom_counts.reshape(-1).tolist() == r["bottom_counts"] and _hx(prof.mean_ts) == r["mean_ts"]
        p = tmp_path / "prof.txt"
        prof.save_text(p)
        assert p.read_text() == r["text"]
    r = trace_golden["planted"]["classify_multi"]
    reps = []
    for i, seed in enumerate(r["seeds"]):
        s2, p2 = S.gen_planted_trace(2, 4, 16, 16, [(0, 0), (1, 3)], 0.85, r["steps"], 128, seed)
        reps.append(compute_stability_report(TopKTrace(f"s{i}", s2, p2), window=8))
    prof = classify_heads(list(reversed(reps)) + [rep], 0.25)  # order-invariant
    assert [list(h) for h in prof.unstable] == r["unstable"] and list(prof.trace_ids) == r["trace_ids"]
    assert prof.bottom_counts.reshape(-1).tolist() == r["bottom_counts"] and _hx(prof.mean_ts) == r["mean_ts"]
    for key, want in trace_golden["planted"]["temporal_8_8"].items():
        l, h = map(int, key.split(","))
        assert float(temporal_stability(tr, HeadId(l, h), 8, 8)).hex() == want


def test_planted_recovery_large_vs_oracle():
    """test_stability.py:157-165 at scale: 8x8 heads, K=64, 256 steps, pool
    1024+ (bitmap of 1040 pages); GPU report == oracle report bit-exactly and
    the classification recovers the planted heads."""
    from paper_2511_00868_b200.stability import classify_heads, compute_stability_report
    from paper_2511_00868_b200.trace import TopKTrace
    planted = [(l, h) for l in range(2) for h in range(8)]
    sel, pools = S.gen_planted_trace(8, 8, 64, 16, planted, 0.9, 256, 1024, 11)
    rep = compute_stability_report(TopKTrace("big", sel, pools), window=32)
    starts, ts, off, deg = S.report(sel, pools, 32, 32)
    assert _hx(rep.ts) == _hx(ts) and _hx(rep.offset_rco) == _hx(off) and rep.degenerate_pairs == deg
    prof = classify_heads([rep], 0.25)
    assert sorted(map(tuple, prof.unstable)) == planted


def test_trace_capture_from_engine(tmp_path):
    """Profiling run: every head scored every step, selections recorded on
    the device inside the step graph; the FXTK trace equals per-step
    snapshots of the selection and round-trips through the container."""
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile, compute_stability_report
    from paper_2511_00868_b200.synthetic import device_normal
    from paper_2511_00868_b200.trace import TraceRecorder, load_trace, save_trace
    B, L, H, G, D, T, K, R, steps = 2, 2, 4, 4, 128, 1000, 8, 4, 20
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25))
    for b in range(B):
        for l in range(L):
            eng.prefill_layer(b, l, device_normal((H, T + 9 * b, D), seed=b * 10 + l),
                              device_normal((H, T + 9 * b, D), seed=b * 10 + l + 5), alloc=(l == 0))
    rec = TraceRecorder(eng, steps, sample_ids=["reqA", "reqB"])
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    snaps, pools = [], []
    for s in range(steps):
        eng.q.normal_(generator=gen)
        eng.k_new.normal_(generator=gen)
        eng.v_new.normal_(generator=gen)
        n_pages = [-(-(n + 1) // 16) for n in eng.seq_host]
        eng.step()
        snaps.append(eng.store.sel[:, :, :, :K].cpu().numpy().astype(np.uint32))
        assert (eng.store.n_sel.cpu().numpy() >= K).all()
        pools.append(n_pages)
    traces = rec.traces()
    assert len(traces) == B and len(eng._graphs) >= 1
    for b, tr in enumerate(traces):
        assert tr.sample_id == ["reqA", "reqB"][b] and tr.n_steps == steps
        assert np.array_equal(tr.selections, np.stack([s[b] for s in snaps]))
        assert tr.pool_sizes.tolist() == [p[b] for p in pools]
        p = tmp_path / f"{tr.sample_id}.fxtk"
        save_trace(tr, p)
        back = load_trace(p)
        assert np.array_equal(back.selections, tr.selections)
        rep = compute_stability_report(tr, window=5, stride=5)
        _, ts, _, _ = S.report(tr.selections, tr.pool_sizes, 5, 5)
        assert _hx(rep.ts) == _hx(ts)
