"""Per-CTA timeline of the head-aligned scoring kernel at config 2
(profiling aid): entry, summary copies issued, streaming done, selection
done (us from the first entry), for one launch with every head due."""
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

B, L, H, G, D, T, K, R = 16, 2, 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25), device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
torch.cuda.synchronize()
st = eng.store
lib = st.lib
lib.fc_debug_score_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(B * H * 4, dtype=torch.int64, device=dev)
res = {}
for rep in range(3):
    buf.zero_()
    lib.fc_debug_score_trace(buf.data_ptr())
    torch.cuda._sleep(10_000_000)
    st.score_select(1, eng.q[1], eng.unstable, R, K, B, force_due=True)
    torch.cuda.synchronize()
    lib.fc_debug_score_trace(None)
tr = buf.view(-1, 4).cpu().numpy().astype(np.float64)
t0 = tr[:, 0].min()
rel = (tr - t0) / 1e3
for i, name in enumerate(["entry", "issued", "streamed", "selected"]):
    res[name] = np.percentile(rel[:, i], [0, 10, 50, 90, 100]).round(2).tolist()
res["stream_body"] = np.percentile(rel[:, 2] - rel[:, 1], [0, 10, 50, 90, 100]).round(2).tolist()
res["select"] = np.percentile(rel[:, 3] - rel[:, 2], [0, 10, 50, 90, 100]).round(2).tolist()
print(json.dumps(res))
