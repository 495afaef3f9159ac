"""Per-warp timeline of the persistent attention kernel (profiling aid):
config-2 shape, one run of NL layers with fc_debug_run_trace.  Prints per
layer the warp-median durations of plan / barrier wait / consumption and the
layer's first-start / last-end spread (us)."""
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

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 8)), 8, 4, 128, 32768, 128, 16
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
lib.fc_debug_run_trace.restype = ctypes.c_int
lib.fc_debug_run_trace.argtypes = [ctypes.c_void_p]
W = 148 * 8
buf = torch.zeros(W * 33 * 8, dtype=torch.int64, device=dev)
out = {}
for nl in (1, L):
    for rep in range(2):
        buf.zero_()
        lib.fc_debug_run_trace(buf.data_ptr())
        torch.cuda._sleep(20_000_000)
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.sparse_decode_layers(0, nl, eng.q[0:nl], eng.out[0:nl], B, max_pages=eng.att_bound,
                                attend_appended=False, first_dep=True)
        b_.record()
        torch.cuda.synchronize()
        lib.fc_debug_run_trace(None)
    tr = buf.view(W, 33, 8).cpu().numpy().astype(np.float64)
    if os.environ.get("DUMP"):
        np.save(os.path.join(os.environ["DUMP"], f"run_trace_nl{nl}.npy"), tr)
    t0 = tr[:, 32, 0].min()
    res = {"event_us": a.elapsed_time(b_) * 1e3,
           "entry_spread_us": (tr[:, 32, 0].max() - t0) / 1e3,
           "first_plan_med_us": float(np.median(tr[:, 32, 1] - tr[:, 32, 0])) / 1e3,
           "exit_last_us": (tr[:, 32, 2].max() - t0) / 1e3, "layers": []}
    for li in range(nl):
        x = tr[:, li]
        res["layers"].append({
            "plan_med": float(np.median(x[:, 1] - x[:, 0])) / 1e3,
            "plan_max": float(np.max(x[:, 1] - x[:, 0])) / 1e3,
            "wait_med": float(np.median(x[:, 2] - x[:, 1])) / 1e3,
            "consume_med": float(np.median(x[:, 3] - x[:, 2])) / 1e3,
            "consume_max": float(np.max(x[:, 3] - x[:, 2])) / 1e3,
            "start_first": (x[:, 2].min() - t0) / 1e3, "start_last": (x[:, 2].max() - t0) / 1e3,
            "end_first": (x[:, 3].min() - t0) / 1e3, "end_last": (x[:, 3].max() - t0) / 1e3,
        })
    out[f"nl{nl}"] = res
print(json.dumps(out, indent=1))
