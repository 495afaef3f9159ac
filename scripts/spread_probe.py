"""Plain-step scored-layer timing at config 2 with the unstable heads spread
over every layer (2 of 8 KV heads per layer; profiling aid): the fused launch
vs scoring + attention as two launches, with the head-aligned or the balanced
scoring kernel, L layers back to back."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200 import _lib  # noqa: E402
from paper_2511_00868_b200.config import HeadId  # noqa: E402
from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 8)), 8, 4, 128, 32768, 128, 16
NU = int(os.environ.get("NU", 2))
dev = torch.device("cuda", 0)
prof = HeadProfile(model_id="spread", n_layers=L, n_heads_per_layer=H, fraction=NU / H,
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
eng.step()  # initial selection; the device step counter is now 2 (a plain step)
torch.cuda.synchronize()
st = eng.store
mp = eng.att_bound
lib = _lib.load()


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


def separate():
    for l in range(L):
        st.score_select(l, eng.q[l], eng.unstable, R, K, B, extra_tokens=1, kv_prefetch=l > 0)
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, extra_tokens=1, attend_appended=False,
                         k_new=eng.k_new[l], v_new=eng.v_new[l], early_unstable=eng.unstable, early_period=R)


def fused():
    for l in range(L):
        plan = eng._mixed_plan(l)
        st.score_attend(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                        kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l],
                        cta_map=plan[0] if plan else None, cluster=plan[1] if plan else 0)


def balanced():
    for l in range(L):
        st.score_attend_balanced(l, eng.q[l], eng.unstable, R, K, eng.out[l], B, extra_tokens=1,
                                 kv_prefetch=l > 0, k_new=eng.k_new[l], v_new=eng.v_new[l])


def score_only():
    for l in range(L):
        st.score_select(l, eng.q[l], eng.unstable, R, K, B, extra_tokens=1, kv_prefetch=l > 0)


def attend_only():
    for l in range(L):
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, extra_tokens=1, attend_appended=False,
                         k_new=eng.k_new[l], v_new=eng.v_new[l], kv_prefetch=l > 0)


import ctypes  # noqa: E402
# parity: the balanced fused launch == balanced scoring + attention, bitwise
lib.fc_debug_score_mode(0)
separate()
torch.cuda.synchronize()
ref = (st.sel.clone(), st.n_sel.clone(), eng.out.clone())
ref_scores = st.scores.clone()
lib.fc_debug_score_mode(-1)
balanced()
torch.cuda.synchronize()
same = (torch.equal(ref[0], st.sel), torch.equal(ref[1], st.n_sel), torch.equal(ref[2], eng.out))
if not all(same):
    dsel = (ref[0] != st.sel).any(-1)
    print("parity: sel heads differing", int(dsel.sum()), "of", dsel.numel(), "n_sel diff", int((ref[1] != st.n_sel).sum()),
          "out max diff", float((ref[2].float() - eng.out.float()).abs().max()),
          "first bad (b,l,h)", dsel.nonzero()[:8].tolist())
    sc = st.scores.view(B * H, -1)[:, :2047]
    rs = ref_scores.view(B * H, -1)[:, :2047]
    bad = (sc != rs)
    for bh in range(12):
        idx = bad[bh].nonzero().flatten()
        print("head", bh, "bad pages", idx.numel(), idx[:3].tolist(), idx[-3:].tolist() if idx.numel() else [])
res = {"balanced_parity": float(all(same)), "grid": float(st.score_attend_balanced_supported(B)),
       "balanced_us": timed(balanced), "fused_us": timed(fused), "attend_only_us": timed(attend_only)}
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=7))

lib.fc_debug_summary_prefetch(ctypes.c_longlong(0))
res["fused_no_prefetch_us"] = timed(fused)
res["balanced_no_prefetch_us"] = timed(balanced)
lib.fc_debug_summary_prefetch(ctypes.c_longlong(-1))
for mode, name in ((1, "head"), (0, "balanced")):
    lib.fc_debug_score_mode(mode)
    res[f"separate_{name}_us"] = timed(separate)
    res[f"score_only_{name}_us"] = timed(score_only)
lib.fc_debug_score_mode(0)
for cps in (1, 2):
    lib.fc_debug_score_ctas_per_sm(cps)
    res[f"separate_balanced_{cps}cps_us"] = timed(separate)
    res[f"score_only_balanced_{cps}cps_us"] = timed(score_only)
lib.fc_debug_score_ctas_per_sm(0)
lib.fc_debug_score_mode(-1)
st.check_errors()
print(json.dumps(res))
