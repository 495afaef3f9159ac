"""Selection traces and head stability on the CPU side:
the oracle is pinned to the reference's outputs on the committed FXTK
fixtures, and the product's host code (FXTK container, text formats,
classification ranking) matches them.  The GPU overlap path is in
test_gpu_stability.py."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, golden_blob
from oracle import stability_oracle as S


def _hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def _corrupt(name, blob, edits):
    if name == "bad_magic":
        return b"NOPE" + blob[4:]
    if name == "bad_version":
        return blob[:4] + struct.pack("<I", 9) + blob[8:]
    if name == "short_header":
        return blob[:10]
    if name == "zero_dim":
        return blob[:12] + struct.pack("<H", 0) + blob[14:]
    if name == "truncated":
        return blob[:-5]
    if name == "trailing":
        return blob + b"\0\0"
    b = bytearray(blob)
    off, val = edits[name]
    struct.pack_into("<I", b, off, val)
    return bytes(b)


# ---- oracle pinned to the reference -------------------------------------------

def test_oracle_generator_and_container_match_reference(trace_golden):
    blob = golden_blob("trace_planted.fxtk")
    sel, pools = S.fxtk_parse(blob)
    c = trace_golden["planted"]["cfg"]
    sel2, pools2 = S.gen_planted_trace(c["L"], c["H"], c["K"], c["page_size"], [tuple(x) for x in c["planted"]],
                                       c["persistence"], c["steps"], c["initial_pool"], c["seed"])
    assert np.array_equal(sel, sel2) and np.array_equal(pools, pools2)
    assert S.fxtk_pack(sel, pools) == blob


@pytest.mark.parametrize("name,window,stride", [("w8", 8, 8), ("w8s4", 8, 4), ("w5s3", 5, 3)])
def test_oracle_report_bit_exact(trace_golden, name, window, stride):
    sel, pools = S.fxtk_parse(golden_blob("trace_planted.fxtk"))
    starts, ts, off, deg = S.report(sel, pools, window, stride)
    r = trace_golden["planted"][name]
    assert list(starts) == r["window_starts"]
    assert _hx(ts) == r["ts"] and _hx(off) == r["offset_rco"] and deg == r["degenerate_pairs"]
    assert S.bottom_counts(ts, 0.25).reshape(-1).tolist() == r["bottom_counts_25"]


def test_oracle_report_degenerate_pools(trace_golden):
    sel, pools = S.fxtk_parse(golden_blob("trace_growth.fxtk"))
    starts, ts, off, deg = S.report(sel, pools, 8, 4)
    r = trace_golden["growth"]
    assert _hx(ts) == r["ts"] and _hx(off) == r["offset_rco"] and deg == r["degenerate_pairs"] > 0


def test_oracle_classify(trace_golden):
    sel, pools = S.fxtk_parse(golden_blob("trace_planted.fxtk"))
    ts = S.report(sel, pools, 8, 8)[1]
    for frac in (0.25, 0.5):
        u, cnt, mean, _ = S.classify([("planted", ts)], frac)
        r = trace_golden["planted"][f"classify_{frac}"]
        assert [list(x) for x in u] == r["unstable"]
        assert cnt.reshape(-1).tolist() == r["bottom_counts"] and _hx(mean) == r["mean_ts"]
    r = trace_golden["planted"]["classify_multi"]
    reps = []
    for i, seed in enumerate(r["seeds"]):
        s2, p2 = S.gen_planted_trace(2, 4, 16, 16, [(0, 0), (1, 3)], 0.85, r["steps"], 128, seed)
        reps.append((f"s{i}", S.report(s2, p2, 8, 8)[1]))
    u, cnt, mean, ids = S.classify(reps + [("planted", ts)], 0.25)
    assert [list(x) for x in u] == r["unstable"] and list(ids) == r["trace_ids"]
    assert cnt.reshape(-1).tolist() == r["bottom_counts"] and _hx(mean) == r["mean_ts"]


def test_oracle_rco_and_load_errors(trace_golden):
    for c in trace_golden["rco_cases"]:
        assert float(S.rco_value(len(set(c["a"]) & set(c["b"])), c["k"], c["pool"])).hex() == c["rco"]
    blob = golden_blob("trace_planted.fxtk")
    for name, want in trace_golden["load_errors"].items():
        with pytest.raises(S.FormatError) as ei:
            S.fxtk_parse(_corrupt(name, blob, trace_golden["load_error_edits"]))
        assert str(ei.value) == want["message"] and ei.value.offset == want["offset"]


# ---- product host code (no GPU needed) -----------------------------------------

def test_trace_container_roundtrip_and_errors(trace_golden, tmp_path):
    from paper_2511_00868_b200.errors import TraceFormatError
    from paper_2511_00868_b200.trace import TopKTrace, load_trace, parse_trace, save_trace
    blob = golden_blob("trace_planted.fxtk")
    tr = load_trace(os.path.join(GOLDEN, "trace_planted.fxtk"))
    assert tr.sample_id == "trace_planted"
    assert (tr.n_steps, tr.n_layers, tr.n_heads_per_layer, tr.k) == (64, 2, 4, 16)
    sel, pools = S.fxtk_parse(blob)
    assert np.array_equal(tr.selections, sel) and np.array_equal(tr.pool_sizes, pools)
    p = tmp_path / "x.fxtk"
    save_trace(tr, p)
    assert p.read_bytes() == blob
    for name, want in trace_golden["load_errors"].items():
        with pytest.raises(TraceFormatError) as ei:
            parse_trace(_corrupt(name, blob, trace_golden["load_error_edits"]), "x")
        assert str(ei.value) == want["message"] and ei.value.offset == want["offset"]
    bad = sel.copy()
    bad[2, 0, 1, 0] = bad[2, 0, 1, 1]
    with pytest.raises(ValueError, match="duplicate"):
        TopKTrace("dup", bad, pools)
    with pytest.raises(ValueError, match="shrink"):
        TopKTrace("shrink", sel, np.concatenate([pools[:5], pools[5:] - 100]))


def test_rco_scalar_and_overlap_helpers(trace_golden, tmp_path):
    from paper_2511_00868_b200.config import HeadId
    from paper_2511_00868_b200.errors import DegeneratePoolError
    from paper_2511_00868_b200.stability import HeadProfile, cross_task_overlap, rco, save_overlap_csv
    for c in trace_golden["rco_cases"]:
        assert float(rco(c["a"], c["b"], c["k"], c["pool"])).hex() == c["rco"]
    assert abs(rco(range(64), range(32, 96), 64, 1024) - 7 / 15) < 1e-12  # test_stability.py:22-27
    with pytest.raises(DegeneratePoolError):
        rco(range(8), range(8), 8, 8)
    with pytest.raises(ValueError):
        rco(range(4), range(8), 8, 64)
    heads = [HeadId(l, h) for l in range(8) for h in range(16)]
    mk = lambda u: HeadProfile(model_id="m", n_layers=8, n_heads_per_layer=16, fraction=0.5,
                               unstable=tuple(u))
    m = cross_task_overlap([mk(heads[:64]), mk(heads[:52] + heads[64:76])])
    assert m[0, 1] == m[1, 0] == 52 / 64 and m[0, 0] == m[1, 1] == 1.0
    save_overlap_csv(m, ["qa", "sum"], tmp_path / "ov.csv")
    assert (tmp_path / "ov.csv").read_text().splitlines()[0] == "task,qa,sum"


def test_profile_text_roundtrip_of_reference_output(trace_golden, tmp_path):
    from paper_2511_00868_b200.stability import HeadProfile
    r = trace_golden["planted"]["classify_0.25"]
    src = tmp_path / "ref.txt"
    src.write_text(r["text"])
    prof = HeadProfile.load_text(src)
    assert [list(h) for h in prof.unstable] == r["unstable"]
    out = tmp_path / "ours.txt"
    prof.save_text(out)
    assert out.read_text() == r["text"]
