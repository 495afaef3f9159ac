"""Per-CTA timeline of fc_score_attend_balanced at config 2 with the unstable
heads spread over every layer (NU of 8 KV heads), L launches back to back;
the last launch's trace (profiling aid).  Slots: entry, staging issued,
released (previous launch complete), staged data landed, phase 1 done,
owner's scores complete, attention start, exit — in us from the release."""
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

B, L, H, G, D, T, K, R = 16, int(os.environ.get("TL", 4)), 8, 4, 128, 32768, 128, 16
NU = int(os.environ.get("NU", 2))
dev = torch.device("cuda", 0)
prof = HeadProfile(model_id="x", n_layers=L, n_heads_per_layer=H, fraction=NU / H,
                   unstable=tuple(HeadId(l, h) for l in range(L) for h in range(NU)))
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=prof, device=dev)
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
lib = st.lib
lib.fc_debug_sa_trace.argtypes = [ctypes.c_void_p]
grid = st.score_attend_balanced_supported(B)


def layers():
    for l in range(L):
        st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                 kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])


st.balanced_helpers = os.environ.get("BAL_WS") == "1"
layers()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    layers()
e1.record()
torch.cuda.synchronize()
print("us per layer", round(e0.elapsed_time(e1) * 1e3 / (10 * L), 2))
sa = torch.zeros(grid * 8, dtype=torch.int64, device=dev)
lib.fc_debug_sa_trace(sa.data_ptr())
torch.cuda._sleep(10_000_000)
layers()
torch.cuda.synchronize()
lib.fc_debug_sa_trace(None)
a = sa.view(-1, 8).cpu().numpy().astype(np.float64)
t0 = a[:, 2].max()  # release: the previous launch complete
n_heads = B * H
role = np.array(["extra"] * grid, dtype=object)
for c in range(grid):
    if c < n_heads:
        role[c] = "owner" if (c % H) < NU else "unscored"
names = ["entry", "issued", "released", "landed", "phase1", "scores_ready", "attn_start", "exit"]
out = {}
for r in ("owner", "unscored", "extra"):
    m = role == r
    out[r] = {n: np.percentile((a[m, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
              for i, n in enumerate(names) if (a[m, i] > 0).all()}
for r, v in out.items():
    print(r, json.dumps(v))
