"""Per-CTA timeline of one config-2 attention launch (profiling aid): sorted
exit times and body durations, to size the load-imbalance tail."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_00868_b200.engine import DecodeEngine
from paper_2511_00868_b200.stability import HeadProfile
from paper_2511_00868_b200.synthetic import device_normal

B, L, H, G, D, T, K, R = int(os.environ.get("B", 16)), 2, 8, 4, 128, 32768, 128, 16
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25))
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(2)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b + l) % 2]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
torch.cuda.synchronize()
st = eng.store
lib = st.lib
lib.fc_debug_attn_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(8192 * 4, dtype=torch.int64, device="cuda")
out = {}
for rep in range(3):
    buf.zero_()
    lib.fc_debug_attn_trace(buf.data_ptr())
    torch.cuda._sleep(5_000_000)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    st.sparse_decode(rep % 2, eng.q[rep % 2], eng.out[rep % 2], B, max_pages=eng.att_bound, attend_appended=False)
    b_.record()
    torch.cuda.synchronize()
    lib.fc_debug_attn_trace(None)
    tr = buf.view(-1, 4).cpu().numpy().astype("float64")
    tr = tr[tr[:, 3] > 0]
    t0 = tr[:, 0].min()
    ex = np.sort((tr[:, 3] - t0) / 1e3)
    body = np.sort((tr[:, 2] - tr[:, 1]) / 1e3)
    iss = np.sort((tr[:, 1] - t0) / 1e3)
    out[rep] = {"event_us": a.elapsed_time(b_) * 1e3, "ctas": len(ex),
                "exit_pcts": [round(float(np.percentile(ex, p)), 2) for p in (0, 5, 25, 50, 75, 95, 100)],
                "issued_pcts": [round(float(np.percentile(iss, p)), 2) for p in (0, 50, 100)],
                "body_pcts": [round(float(np.percentile(body, p)), 2) for p in (0, 5, 25, 50, 75, 95, 100)],
                "mean_exit": round(float(ex.mean()), 2)}
print(json.dumps(out))
