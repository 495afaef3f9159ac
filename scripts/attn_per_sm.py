"""Per-SM attention bandwidth with one CTA per head at low occupancy
(profiling aid): fc_sparse_decode n_ctas=1 over B*8 heads at 32k context,
K = 128 pages, and the scoring-only launch for the same heads."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

res = {}
for B in (1, 4, 16):
    L, H, G, D, T, K, R = 1, 8, 4, 128, 32768, 128, 16
    eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                       topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 1.0))
    k, v = device_normal((H, T, D), seed=1), device_normal((H, T, D), seed=2)
    for b in range(B):
        eng.prefill_layer(b, 0, k, v, alloc=True)
    eng.q.normal_()
    eng.step()
    torch.cuda.synchronize()
    st = eng.store
    out = torch.zeros_like(eng.out[0])

    def timed(fn, n=20):
        fn()
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b_.record()
        b_.synchronize()
        return a.elapsed_time(b_) / n * 1e3

    heads = B * H
    att_bytes = heads * (K + 1) * st.page_bytes
    t1 = timed(lambda: st.sparse_decode(0, eng.q[0], out, B, max_pages=eng.att_bound, extra_tokens=1,
                                        attend_appended=False, n_ctas=1))
    ts = timed(lambda: st.score_select(0, eng.q[0], eng.unstable, R, K, B, force_due=True, extra_tokens=1))
    summ = heads * (T // 16) * 2 * D * 2
    res[f"B{B}"] = {"heads": heads, "attn_1cta_us": round(t1, 2),
                    "attn_GBps_per_cta": round(att_bytes / heads / (t1 * 1e3), 1),
                    "score_us": round(ts, 2), "score_GBps_per_head": round(summ / heads / (ts * 1e3), 1)}
    del eng
    torch.cuda.empty_cache()
print(json.dumps(res))

# timeline of one isolated one-CTA-per-head launch at B = 4 (warp 0 of each CTA)
import ctypes  # noqa: E402
import numpy as np  # noqa: E402

B = 4
eng = DecodeEngine(batch=B, layers=1, kv_heads=8, group=4, head_dim=128, ctx_cap_tokens=32768 + 64,
                   topk_pages=128, rerank_period=16, profile=HeadProfile.first_n(1, 8, 1.0))
k, v = device_normal((8, 32768, 128), seed=1), device_normal((8, 32768, 128), seed=2)
for b in range(B):
    eng.prefill_layer(b, 0, k, v, alloc=True)
eng.q.normal_()
eng.step()
torch.cuda.synchronize()
st = eng.store
out = torch.zeros_like(eng.out[0])
lib = st.lib
lib.fc_debug_attn_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(64 * 4, dtype=torch.int64, device="cuda")
tl = {}
for rep in range(3):
    buf.zero_()
    lib.fc_debug_attn_trace(buf.data_ptr())
    torch.cuda._sleep(5_000_000)
    st.sparse_decode(0, eng.q[0], out, B, max_pages=eng.att_bound, extra_tokens=1, attend_appended=False, n_ctas=1)
    torch.cuda.synchronize()
    lib.fc_debug_attn_trace(None)
tr = buf.view(-1, 4).cpu().numpy().astype(np.float64)
tr = tr[tr[:, 3] > 0]
t0 = tr[:, 0].min()
for i, name in enumerate(["entry", "issued", "loop_done", "exit"]):
    tl[name] = np.percentile((tr[:, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
tl["prologue"] = np.percentile((tr[:, 1] - tr[:, 0]) / 1e3, [0, 50, 100]).round(2).tolist()
tl["loop"] = np.percentile((tr[:, 2] - tr[:, 1]) / 1e3, [0, 50, 100]).round(2).tolist()
tl["merge"] = np.percentile((tr[:, 3] - tr[:, 2]) / 1e3, [0, 50, 100]).round(2).tolist()
print(json.dumps(tl))
