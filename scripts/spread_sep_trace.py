"""Timeline of a spread-profile scored layer run as two launches (profiling
aid): the balanced scoring kernel (CTAs per SM = CPS) then the attention
kernel with early_unstable, L layers back to back; the last layer's per-CTA
entry / exit of both kernels (attention split into heads scored this step
and the others), in us from the scoring launch's first CTA."""
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

B, L, H, G, D, T, K, R = 16, 4, 8, 4, 128, 32768, 128, 16
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
assert int(st.step.item()) % R != 0
lib = st.lib
for f in ("fc_debug_attn_trace", "fc_debug_score_trace"):
    getattr(lib, f).argtypes = [ctypes.c_void_p]
mp = eng.att_bound


def layers():
    for l in range(L):
        st.score_select(l, eng.q[l], eng.unstable, R, K, B, extra_tokens=1, kv_prefetch=l > 0)
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, extra_tokens=1, attend_appended=False,
                         k_new=eng.k_new[l], v_new=eng.v_new[l], early_unstable=eng.unstable, early_period=R)


res = {}
for mode, cps in ((0, 1), (0, 2), (0, 0), (1, 0)):
    lib.fc_debug_score_mode(mode)
    lib.fc_debug_score_ctas_per_sm(cps)
    at = torch.zeros(B * H * 4, dtype=torch.int64, device=dev)
    sc = torch.zeros(148 * 8 * 4, dtype=torch.int64, device=dev)
    layers()
    torch.cuda.synchronize()
    lib.fc_debug_attn_trace(at.data_ptr())
    lib.fc_debug_score_trace(sc.data_ptr())
    torch.cuda._sleep(10_000_000)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    layers()
    b_.record()
    torch.cuda.synchronize()
    lib.fc_debug_attn_trace(None)
    lib.fc_debug_score_trace(None)
    A = at.view(-1, 4).cpu().numpy().astype(np.float64)
    C = sc.view(-1, 4).cpu().numpy().astype(np.float64)
    C = C[C[:, 0] > 0]
    t0 = C[:, 0].min()
    scored = np.array([(i % H) < NU for i in range(B * H)])
    pct = lambda x: np.percentile((x - t0) / 1e3, [0, 50, 100]).round(2).tolist()  # noqa: E731
    r = {"layer_us": round(a.elapsed_time(b_) * 1e3 / L, 2),
         "score_entry": pct(C[:, 0]), "score_exit": pct(C[:, 3][C[:, 3] > 0]),
         "n_score_ctas": int(len(C))}
    for name, m in (("att_scored", scored), ("att_unscored", ~scored)):
        r[name + "_entry"] = pct(A[m, 0])
        r[name + "_loop"] = pct(A[m, 2])
        r[name + "_exit"] = pct(A[m, 3])
    res[f"mode{mode}_cps{cps}"] = r
lib.fc_debug_score_mode(-1)
lib.fc_debug_score_ctas_per_sm(0)
st.check_errors()
for k, v in res.items():
    print(k, json.dumps(v))
