"""One fc_sparse_decode launch, one CTA per head, B=4 (32 heads) at 32k
context, K=128 (for an ncu capture of the low-occupancy per-CTA rate)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 4, 1, 8, 4, 128, 32768, 128, 16
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 1.0))
k, v = device_normal((H, T, D), seed=1), device_normal((H, T, D), seed=2)
for b in range(B):
    eng.prefill_layer(b, 0, k, v, alloc=True)
eng.q.normal_()
eng.step()
torch.cuda.synchronize()
out = torch.zeros_like(eng.out[0])
for _ in range(3):
    eng.store.sparse_decode(0, eng.q[0], out, B, max_pages=eng.att_bound, extra_tokens=1, attend_appended=False,
                            n_ctas=1)
torch.cuda.synchronize()
