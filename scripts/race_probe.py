"""Racecheck driver (profiling aid): one launch of the head-aligned scoring
kernel or of the fused kernel (one CTA per head) at a context long enough
that the scoring ring refills.  argv[1]: score | fused | mixed."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200 import _lib  # noqa: E402
from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, H, G, D, T, K = 2, 8, 4, 128, 6000, 32
eng = DecodeEngine(batch=B, layers=1, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=4, profile=HeadProfile.first_n(1, H, 0.25))
for b in range(B):
    eng.prefill_layer(b, 0, device_normal((H, T, D), seed=b), device_normal((H, T, D), seed=9 + b), alloc=True)
st = eng.store
q = device_normal(tuple(eng.q[0].shape), seed=7)
out = torch.zeros_like(eng.out[0])
lib = _lib.load()
lib.fc_debug_score_mode.argtypes = [ctypes.c_int]
mode = sys.argv[1]
if mode == "score":
    lib.fc_debug_score_mode(1)
    st.score_select(0, q, eng.unstable, 4, K, B, force_due=True, extra_tokens=1)
elif mode == "fused":
    lib.fc_debug_score_mode(1)
    st.score_attend(0, q, eng.unstable, 4, K, out, B, force_due=True, extra_tokens=1)
else:
    m = []
    for b in range(B):
        for h in range(H):
            m += [(b * H + h) | (1 << 30)]
    t = torch.tensor(m, dtype=torch.int32, device="cuda")
    st.score_attend(0, q, eng.unstable, 4, K, out, B, force_due=True, extra_tokens=1, cta_map=t, cluster=2)
torch.cuda.synchronize()
st.check_errors()
print("ok", mode)
