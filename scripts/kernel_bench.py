"""Per-kernel timing at config 2 (profiling aid, not the bench line): each
kernel launched back to back over the 32 layers (distinct data, > L2), one
event pair around the 32 launches, best of 3.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = (int(os.environ.get("B", 16)), int(os.environ.get("L", 32)), 8, 4, 128,
                          int(os.environ.get("T", 32768)), 128, 16)
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25), device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
del srcs
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
torch.cuda.synchronize()
st = eng.store


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        for layer in range(L):
            fn(layer)
        b_.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b_) * 1e3 / L)
    return best


att_bytes = sum(eng.attention_bytes(l) for l in range(L)) / L
sc_bytes = eng.scoring_bytes(0, 1)
import ctypes  # noqa: E402
from paper_2511_00868_b200 import _lib  # noqa: E402
lib = _lib.load()
lib.fc_debug_score_mode.argtypes = [ctypes.c_int]


def moded(mode, fn):
    def run(layer):
        fn(layer)
    lib.fc_debug_score_mode(mode)
    try:
        return timed(run)
    finally:
        lib.fc_debug_score_mode(-1)


res = {
    "attn_us": timed(lambda l: st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=eng.att_bound,
                                                 attend_appended=False)),
    "score_select_us": timed(lambda l: st.score_select(l, eng.q[l], eng.unstable, R, K, B, force_due=True)),
    "score_select_bal_us": moded(0, lambda l: st.score_select(l, eng.q[l], eng.unstable, R, K, B, force_due=True)),
    "score_select_head_us": moded(1, lambda l: st.score_select(l, eng.q[l], eng.unstable, R, K, B, force_due=True)),
    "unstable_bal_us": moded(0, lambda l: st.score_select(l, eng.q[l], eng.unstable, R, K, B)),
    "unstable_head_us": moded(1, lambda l: st.score_select(l, eng.q[l], eng.unstable, R, K, B)),
    "score_only_us": timed(lambda l: st.score_pages(l, eng.q[l], B, extra_tokens=1)),
}
res["attn_GBs"] = att_bytes / (res["attn_us"] * 1e-6) / 1e9
res["score_GBs"] = sc_bytes / (res["score_only_us"] * 1e-6) / 1e9
res["score_select_GBs"] = sc_bytes / (res["score_select_us"] * 1e-6) / 1e9
print(json.dumps(res))
