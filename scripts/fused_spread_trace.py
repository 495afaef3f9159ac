"""Fused scored layer at config 2 with a spread profile (2 of 8 KV heads of
every layer unstable): per-CTA scoring timeline of the due heads and launch
times of the variants (profiling aid)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_00868_b200.config import HeadId  # noqa: E402
from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 16, 2, 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
prof = HeadProfile(model_id="x", n_layers=L, n_heads_per_layer=H, fraction=0.25,
                   unstable=tuple(HeadId(l, h) for l in range(L) for h in range(2)))
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=prof, device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
eng.step()
torch.cuda.synchronize()
st = eng.store
assert int(st.step.item()) % R != 0
lib = st.lib
res = {}


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return round(a.elapsed_time(b) / n * 1e3, 2)


out = torch.zeros_like(eng.out[1])
res["fused_plain_us"] = timed(lambda: st.score_attend(1, eng.q[1], eng.unstable, R, K, out, B, extra_tokens=1))
res["fused_all_due_us"] = timed(lambda: st.score_attend(1, eng.q[1], eng.unstable, R, K, out, B, force_due=True,
                                                        extra_tokens=1))
res["attn_only_us"] = timed(lambda: st.sparse_decode(1, eng.q[1], out, B, max_pages=eng.att_bound, extra_tokens=1,
                                                     attend_appended=False, n_ctas=1))
res["attn_split_us"] = timed(lambda: st.sparse_decode(1, eng.q[1], out, B, max_pages=eng.att_bound, extra_tokens=1,
                                                      attend_appended=False))
res["score_plain_us"] = timed(lambda: st.score_select(1, eng.q[1], eng.unstable, R, K, B, extra_tokens=1))
def pair():
    st.score_select(1, eng.q[1], eng.unstable, R, K, B, extra_tokens=1)
    st.sparse_decode(1, eng.q[1], out, B, max_pages=eng.att_bound, extra_tokens=1, attend_appended=False,
                     early_unstable=eng.unstable, early_period=R)


def pair_no_early():
    st.score_select(1, eng.q[1], eng.unstable, R, K, B, extra_tokens=1)
    st.sparse_decode(1, eng.q[1], out, B, max_pages=eng.att_bound, extra_tokens=1, attend_appended=False)


def mapped(S, due_heads, split_all, force=False):
    m, rest = [], []
    for b in range(B):
        for h in range(H):
            bh = b * H + h
            if h in due_heads:
                m += [bh] * S
            elif split_all:
                rest += [bh] * S
            else:
                rest.append(bh | (1 << 30))
    m += rest
    m += [-1] * (-len(m) % S)
    t = torch.tensor(m, dtype=torch.int32, device=dev)
    return timed(lambda: st.score_attend(1, eng.q[1], eng.unstable, R, K, out, B, extra_tokens=1, force_due=force,
                                         cta_map=t, cluster=S))


for S in (2, 3, 4):
    res[f"map_plain_split_all_S{S}_us"] = mapped(S, (0, 1), True)
    res[f"map_alldue_split_all_S{S}_us"] = mapped(S, tuple(range(H)), True, force=True)
res["map_plain_S2_stable_alone_us"] = mapped(2, (0, 1), False)
res["pair_early_us"] = timed(pair)
res["pair_us"] = timed(pair_no_early)
lib.fc_debug_score_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(B * H * 4, dtype=torch.int64, device=dev)
buf.zero_()
lib.fc_debug_score_trace(buf.data_ptr())
torch.cuda._sleep(10_000_000)
st.score_attend(1, eng.q[1], eng.unstable, R, K, out, B, extra_tokens=1)
torch.cuda.synchronize()
lib.fc_debug_score_trace(None)
tr = buf.view(-1, 4).cpu().numpy().astype(np.float64)
due = tr[:, 2] > 0
t0 = tr[:, 0][tr[:, 0] > 0].min()
rel = (tr[due] - t0) / 1e3
for i, name in enumerate(["entry", "issued", "streamed", "selected"]):
    res[name] = np.percentile(rel[:, i], [0, 50, 100]).round(2).tolist()
res["stream_body"] = np.percentile(rel[:, 2] - rel[:, 1], [0, 50, 100]).round(2).tolist()
res["select"] = np.percentile(rel[:, 3] - rel[:, 2], [0, 50, 100]).round(2).tolist()
res["n_due_ctas"] = int(due.sum())
print(json.dumps(res))
