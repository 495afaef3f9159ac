"""Plain-step and rerank-step time at config 2 with and without early head
start (profiling aid).  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = int(os.environ.get("B", 16)), 32, 8, 4, 128, 32768, 128, 16
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 256,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25))
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
del srcs
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
eng.capture_graphs()
res = {}
for early in (False, True, False, True):
    eng.early_heads = early
    eng._graphs.clear()
    eng.capture_graphs()
    plain, rr = [], []
    for i in range(48):
        rerank = eng.is_rerank_step()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.step()
        b_.record()
        torch.cuda.synchronize()
        (rr if rerank else plain).append(a.elapsed_time(b_))
    plain.sort()
    res[f"early={early}"] = {"plain_p50_ms": plain[len(plain) // 2], "rerank_ms": sorted(rr)}
print(json.dumps(res))
