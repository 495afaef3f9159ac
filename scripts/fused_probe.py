"""Scored-layer timing at config 2 (profiling aid): score_select +
sparse_decode vs fc_score_attend, every head due, 8 layers back to back."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 8)), 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 1.0), device=dev)
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
mp = eng.att_bound


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        fn()
        b_.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b_) * 1e3)
    return best / L


def separate():
    for l in range(L):
        st.score_select(l, eng.q[l], eng.unstable, R, K, B, force_due=True, extra_tokens=1, kv_prefetch=l > 0)
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, extra_tokens=1, attend_appended=False,
                         k_new=eng.k_new[l], v_new=eng.v_new[l])


def fused():
    for l in range(L):
        st.score_attend(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, force_due=True, extra_tokens=1,
                        kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])


def score_only():
    for l in range(L):
        st.score_select(l, eng.q[l], eng.unstable, R, K, B, force_due=True, extra_tokens=1, kv_prefetch=l > 0)


res = {"separate_us": timed(separate), "fused_us": timed(fused), "score_only_us": timed(score_only)}
st.check_errors()
print(json.dumps(res))
