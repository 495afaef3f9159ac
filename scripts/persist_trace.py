"""Per-CTA timeline of the per-head persistent attention kernel (profiling
aid): one run of NL layers at batch B (env), config-2 shape otherwise.
Prints per layer the CTA-median of (barrier+q wait, consume, merge+publish)
and the layer's consumption start spread (us)."""
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

B, L, H, G, D, T, K, R = int(os.environ.get("B", 8)), int(os.environ.get("L", 8)), 8, 4, 128, 32768, 128, 16
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
lib.fc_debug_persist_trace.argtypes = [ctypes.c_void_p]
S = st.run_split(B, eng.att_bound)
grid = B * H * S
buf = torch.zeros(grid * 33 * 4, dtype=torch.int64, device=dev)
for rep in range(2):
    buf.zero_()
    lib.fc_debug_persist_trace(buf.data_ptr())
    torch.cuda._sleep(10_000_000)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st.sparse_decode_layers(0, L, eng.q, eng.out, B, max_pages=eng.att_bound, attend_appended=False,
                            first_dep=True)
    b_.record()
    torch.cuda.synchronize()
    lib.fc_debug_persist_trace(None)
tr = buf.view(grid, 33, 4).cpu().numpy().astype(np.float64)
t0 = tr[:, 32, 0].min()
out = {"S": S, "grid": grid, "event_us": a.elapsed_time(b_) * 1e3, "layers": []}
for li in range(L):
    x = tr[:, li]
    row = {"wait": float(np.median(x[:, 1] - x[:, 0])) / 1e3,
           "consume": float(np.median(x[:, 2] - x[:, 1])) / 1e3,
           "consume_max": float(np.max(x[:, 2] - x[:, 1])) / 1e3,
           "start_spread": float(x[:, 1].max() - x[:, 1].min()) / 1e3,
           "start": float(np.median(x[:, 1]) - t0) / 1e3}
    if li + 1 < L:
        row["merge_publish"] = float(np.median(x[:, 3] - x[:, 2])) / 1e3
        row["merge_publish_max"] = float(np.max(x[:, 3] - x[:, 2])) / 1e3
    out["layers"].append({k: round(v, 2) for k, v in row.items()})
print(json.dumps(out))
