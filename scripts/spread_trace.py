"""Per-CTA timeline of the fused scored layer at config 2 with the unstable
heads spread over every layer (2 of 8 KV heads), L launches back to back as
in a plain step (profiling aid).  The timeline is the LAST launch's (every
launch overwrites the trace): entry, selection visible, attention done and
exit per CTA, split into scored and unscored CTAs; with and without the
next-layer summary warm-up."""
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
lib.fc_debug_sa_trace.argtypes = [ctypes.c_void_p]
lib.fc_debug_score_trace.argtypes = [ctypes.c_void_p]
lib.fc_debug_summary_prefetch.argtypes = [ctypes.c_longlong]


WARM = False
BAL = os.environ.get('BAL') == '1'


def layers():
    for l in range(L):
        if WARM and l == L - 1:  # the last layer's due summaries read just before: L2-resident
            st.score_select(l, eng.q[l], eng.unstable, R, K, B, extra_tokens=1)
        if BAL:
            st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                     kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])
        else:
            st.score_attend(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1, kv_prefetch=l > 0,
                            k_new=eng.k_new[l], v_new=eng.v_new[l])


res = {}
for pf in (-1, 0, 1):
    WARM = pf == 1
    lib.fc_debug_summary_prefetch(0 if WARM else pf)
    sa = torch.zeros(148 * 4, dtype=torch.int64, device=dev)
    sc = torch.zeros(B * H * 4, dtype=torch.int64, device=dev)
    layers()
    torch.cuda.synchronize()
    lib.fc_debug_sa_trace(sa.data_ptr())
    lib.fc_debug_score_trace(sc.data_ptr())
    torch.cuda._sleep(10_000_000)
    layers()
    torch.cuda.synchronize()
    lib.fc_debug_sa_trace(None)
    lib.fc_debug_score_trace(None)
    a = sa.view(-1, 4).cpu().numpy().astype(np.float64)[:B * H]
    extra = sa.view(-1, 4).cpu().numpy().astype(np.float64)[B * H:]
    c = sc.view(-1, 4).cpu().numpy().astype(np.float64)
    t0 = a[:, 0].min()
    scored = np.array([(i % H) < NU for i in range(B * H)])
    r = {}
    for name, m in (("scored", scored), ("unscored", ~scored)):
        rel = (a[m] - t0) / 1e3
        r[name] = {k: np.percentile(rel[:, i], [0, 50, 100]).round(2).tolist()
                   for i, k in enumerate(["entry", "selected", "attended", "exit"])}
    if BAL:
        r["extra_ctas"] = {k: np.percentile((extra[:, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
                           for i, k in enumerate(["entry", "scored"])}
        res["warm" if WARM else "prefetch" if pf else "no_prefetch"] = r
        continue
    cr = (c[scored] - t0) / 1e3
    r["scored"].update({k: np.percentile(cr[:, i], [0, 50, 100]).round(2).tolist()
                        for i, k in enumerate(["s_entry", "s_issued", "s_streamed", "s_selected"])})
    res["warm" if WARM else "prefetch" if pf else "no_prefetch"] = r
lib.fc_debug_summary_prefetch(-1)
st.check_errors()
print(json.dumps(res, indent=1))
