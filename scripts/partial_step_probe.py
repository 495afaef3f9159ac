"""Whole-step timing with staggered request phases (profiling aid): config 2
(32 layers, fixture mask u = 0.25, 16 rows at 32k), row b starts at its own
t = 1 + b, so every step has one row at its rerank boundary.  Step time with
the step graph and eagerly; the per-layer kind of launch; then the balanced
launch timeline of the last layer (g_sa_trace)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 32)), 8, 4, 128, 32768, 128, 16
U = float(os.environ.get("U", 0.25))
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 256,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, U), device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
del srcs
if os.environ.get("PHASES", "staggered") == "staggered":
    for b in range(B):
        eng.set_row_step(b, 1 + b % int(os.environ.get("PHASE_MOD", R)))
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
kg = torch.Generator(device="cuda")
kg.manual_seed(5)
_step = eng.step


def fresh_step(**kw):  # a distinct appended token every step
    eng.k_new.normal_(generator=kg)
    eng.v_new.normal_(generator=kg)
    return _step(**kw)


eng.step = fresh_step
for _ in range(4):
    eng.step()
torch.cuda.synchronize()


def timed(fn, n=16):
    ts = []
    for _ in range(n):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(5_000_000)
        a.record()
        fn()
        b_.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b_) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


res = {"kind": eng.step_kind(), "graph_step_us": timed(lambda: eng.step()),
       "graph_step_us_2": timed(lambda: eng.step()),
       "eager_step_us": timed(lambda: eng.step(use_graph=False)),
       "graph_step_us_3": timed(lambda: eng.step())}
import time  # noqa: E402
torch.cuda.synchronize()
torch.cuda._sleep(200_000_000)
h0 = time.perf_counter()
a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a0.record()
for _ in range(64):
    eng.step()
h1 = time.perf_counter()
a1.record()
torch.cuda.synchronize()
res["host_us_per_step"] = (h1 - h0) / 64 * 1e6
res["gpu_us_per_step_64"] = a0.elapsed_time(a1) * 1e3 / 64


def b2b(n, gap=0, nofill=False):
    saved = eng._fill_partial_maps
    if nofill:
        eng._fill_partial_maps = lambda: None
    torch.cuda.synchronize()
    torch.cuda._sleep(100_000_000)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    e[0].record()
    for i in range(n):
        if gap:
            torch.cuda._sleep(gap)
        eng.step()
        e[i + 1].record()
    torch.cuda.synchronize()
    eng._fill_partial_maps = saved
    seq = [round(e[i].elapsed_time(e[i + 1]) * 1e3) for i in range(n)]
    ts = sorted(seq)
    return [round(ts[0]), round(ts[len(ts) // 2]), round(ts[-1])] + ([seq] if os.environ.get("SEQ") else [])


for sl in (2_000_000, 200_000, 20_000):
    res[f"single_after_sleep_{sl}"] = round(timed(lambda: eng.step()) if sl == 5_000_000 else 0)
    ts = []
    for _ in range(8):
        a_, b__ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(sl)
        a_.record()
        eng.step()
        b__.record()
        torch.cuda.synchronize()
        ts.append(a_.elapsed_time(b__) * 1e3)
    res[f"single_after_sleep_{sl}"] = round(sorted(ts)[4])
res["b2b_32"] = b2b(32)
res["b2b_32_gap"] = b2b(32, gap=20000)
res["b2b_32_nofill"] = b2b(32, nofill=True)
lib = eng.store.lib
lib.fc_debug_sa_trace.argtypes = [ctypes.c_void_p]
grid = eng.store.score_attend_balanced_supported(B)
sa = torch.zeros(grid * 8, dtype=torch.int64, device=dev)
lib.fc_debug_sa_trace(sa.data_ptr())
if os.environ.get("TRACE_B2B", "1") == "1":
    for _ in range(8):
        eng.step()
else:
    torch.cuda._sleep(5_000_000)
    eng.step()
torch.cuda.synchronize()
lib.fc_debug_sa_trace(None)
a = sa.view(-1, 8).cpu().numpy().astype(np.float64)
t0 = a[:, 2].max()
due_row = [b for b in range(B) if (eng.t - 1 + eng.phase[b]) % R == 0]
role = np.array(["extra"] * grid, dtype=object)
for c in range(min(grid, B * H)):
    role[c] = "owner" if c // H in due_row else "unscored"
for c in range(B * H, grid):
    if a[c, 5] > 0:
        role[c] = "helper"
names = ["entry", "issued", "released", "landed", "phase1", "scores_ready", "attn_start", "exit"]
tr = {}
for r in ("owner", "unscored", "helper", "extra"):
    m = role == r
    if m.any():
        tr[r] = {n: np.percentile((a[m, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
                 for i, n in enumerate(names) if (a[m, i] > 0).all()}
res["due_rows"] = due_row
res["balanced_trace_last_layer"] = tr
eng.store.check_errors()
print(json.dumps(res))

# the due row's score rows after the last step (what the owners selected from)
if os.environ.get("SCORES"):
    sc = eng.store.scores.view(B, H, -1).float().cpu().numpy()
    n_pages = (int(eng.store.seq_len.max().item()) + 1 + 15) // 16
    np.save("gpurun_out/due_scores.npy", sc[due_row[0], :, :n_pages - 1])
    for b in due_row[:1]:
        for h in range(2):
            row = sc[b, h, :n_pages - 1]
            lo, hi = row.min(), row.max()
            bins = np.minimum(((row - lo) * (2048 / (hi - lo))).astype(int), 2047)
            cnt = np.bincount(bins, minlength=2048)
            print(json.dumps({"b": b, "h": h, "min": float(lo), "max": float(hi), "p50": float(np.median(row)),
                              "max_bin": int(cnt.max()), "nonempty_bins": int((cnt > 0).sum()),
                              "top_k_bin_count": int(cnt[np.searchsorted(np.cumsum(cnt[::-1]), 127)])}))
