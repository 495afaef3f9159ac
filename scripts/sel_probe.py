import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2511_00868_b200.engine import DecodeEngine
from paper_2511_00868_b200.stability import HeadProfile
from paper_2511_00868_b200.synthetic import device_normal
B, L, H, G, D, T, K, R = 16, 1, 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.0), device=dev)
k, v = device_normal((H, T, D), seed=1), device_normal((H, T, D), seed=2)
for b in range(B):
    eng.prefill_layer(b, 0, k, v, alloc=True)
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()
for b in range(B):
    eng.set_row_step(b, R if b == 0 else 1 + b % (R - 1))
eng.store.per_row = True
torch.cuda.synchronize()
print("=== balanced", flush=True)
st = eng.store
st.score_attend_balanced(0, eng.q[0], eng.unstable, R, K, eng.out[0], B, extra_tokens=1, kv_prefetch=False,
                         k_new=eng.k_new[0], v_new=eng.v_new[0])
torch.cuda.synchronize()
print("=== fused one CTA per head (all due)", flush=True)
st.score_attend(0, eng.q[0], eng.unstable, R, K, eng.out[0], B, force_due=True, extra_tokens=1)
torch.cuda.synchronize()
