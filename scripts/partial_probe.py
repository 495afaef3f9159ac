"""Partial-step layer timing at config 2 (profiling aid): all heads stable,
one row (of 16) at its rerank boundary, so 8 of the layer's 128 heads are
scored.  Per layer, L layers back to back: attention only (a plain layer),
the balanced launch, and the fused map launch with the due row's heads in
clusters of S CTAs (the others one CTA each)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 8)), 8, 4, 128, 32768, 128, 16
NDUE = int(os.environ.get("NDUE", 1))
dev = torch.device("cuda", 0)
prof = HeadProfile.first_n(L, H, 0.0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=prof, device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(4)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b * L + l) % 4]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
del srcs
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()  # initial selection; the upcoming global step is 2
for b in range(B):  # rows 0..NDUE-1 at their boundary at step 2
    eng.set_row_step(b, R if b < NDUE else 1 + b % (R - 1))
eng.store.per_row = True
torch.cuda.synchronize()
st = eng.store
mp = eng.att_bound


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(20_000_000)
        a.record()
        fn()
        b_.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b_) * 1e3)
    return best / L


def attend_only():
    for l in range(L):
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, extra_tokens=1, attend_appended=False,
                         k_new=eng.k_new[l], v_new=eng.v_new[l], kv_prefetch=l > 0)


def balanced():
    for l in range(L):
        st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                 kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])


def fused_map(m, S):
    def f():
        for l in range(L):
            st.score_attend(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                            kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l], cta_map=m, cluster=S)
    return f


def fused_uniform():
    for l in range(L):
        st.score_attend(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                        kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])


res = {"attend_only_us": timed(attend_only), "balanced_us": timed(balanced), "fused_uniform_us": timed(fused_uniform)}
scored = {(b, h) for b in range(NDUE) for h in range(H)}
for S in (2, 3, 4):
    n_ctas = (len(scored) + -(-(B * H - len(scored)) // S)) * S
    if n_ctas > 148 or not st.score_attend_map_fits(n_ctas, S):
        res[f"map_S{S}"] = "no fit"
        continue
    m = st.cluster_map_pairs(B, scored, S, n_ctas).to(dev)
    res[f"map_S{S}_us"] = timed(fused_map(m, S))
res["plan"] = eng._partial_plan(0)[1] if eng._partial_plan(0) else None
st.check_errors()
print(json.dumps(res))

# per-CTA timeline of the map launch (S = 2): entry, attention start (the
# selection visible), attention done, exit — us from the earliest entry
if os.environ.get("TRACE", "1") == "1":
    import ctypes
    import numpy as np
    S = int(os.environ.get("TS", 3))
    n_ctas = (len(scored) + -(-(B * H - len(scored)) // S)) * S
    mh = st.cluster_map_pairs(B, scored, S, n_ctas)
    m = mh.to(dev)
    lib = st.lib
    lib.fc_debug_sa_trace.argtypes = [ctypes.c_void_p]
    fused_map(m, S)()
    torch.cuda.synchronize()
    sa = torch.zeros(n_ctas * 4, dtype=torch.int64, device=dev)
    lib.fc_debug_score_trace.argtypes = [ctypes.c_void_p]
    sc = torch.zeros(n_ctas * 4, dtype=torch.int64, device=dev)
    lib.fc_debug_sa_trace(sa.data_ptr())
    lib.fc_debug_score_trace(sc.data_ptr())
    torch.cuda._sleep(10_000_000)
    fused_map(m, S)()
    torch.cuda.synchronize()
    lib.fc_debug_sa_trace(None)
    lib.fc_debug_score_trace(None)
    c4 = sc.view(-1, 4).cpu().numpy().astype(np.float64)
    a = sa.view(-1, 4).cpu().numpy().astype(np.float64)
    mm = mh.numpy()
    t0 = a[mm >= 0, 0].min()
    roles = {"scored": (mm >= 0) & (mm & (1 << 30) == 0), "alone": (mm >= 0) & (mm & (1 << 30) != 0)}
    tr = {}
    for r, sel in roles.items():
        tr[r] = {n: np.percentile((a[sel, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
                 for i, n in enumerate(["entry", "attn_start", "attn_done", "exit"]) if (a[sel, i] > 0).all()}
        tr[r].update({n: np.percentile((c4[sel, i] - t0) / 1e3, [0, 50, 100]).round(2).tolist()
                      for i, n in enumerate(["s_entry", "s_released", "s_streamed", "s_selected"])
                      if (c4[sel, i] > 0).all()})
    print(json.dumps(tr))
    late = np.flatnonzero(roles["alone"] & ((a[:, 1] - t0) / 1e3 > 70))
    print("late alone CTAs", late.tolist(), ((a[late, :] - t0) / 1e3).round(1).tolist(),
          "their heads", [int(mm[i] & 0xffff) for i in late])
