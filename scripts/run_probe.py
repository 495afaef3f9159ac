"""Attention timing at config 2 (profiling aid, not the bench line): the
per-layer kernel (fc_sparse_decode, 32 launches) vs the persistent run
kernel (fc_sparse_decode_layers) as 32 single-layer launches, 4 runs of 8
and one run of 32; plus whole engine steps with each.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

B, L, H, G, D, T, K, R = int(os.environ.get("B", 16)), int(os.environ.get("L", 32)), 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25), device=dev)
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
    return best


def per_layer():
    for l in range(L):
        st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=mp, attend_appended=False,
                         kv_prefetch=l > 0)


def runs(n):
    def f():
        for l0 in range(0, L, n):
            st.sparse_decode_layers(l0, n, eng.q[l0:l0 + n], eng.out[l0:l0 + n], B, max_pages=mp,
                                    attend_appended=False, first_dep=(l0 == 0))
    return f


res = {}
att_bytes = sum(eng.attention_bytes(l) for l in range(L))
import ctypes  # noqa: E402
st.lib.fc_debug_run_mode.argtypes = [ctypes.c_int]


def moded(mode, fn):
    def f():
        st.lib.fc_debug_run_mode(mode)
        try:
            fn()
        finally:
            st.lib.fc_debug_run_mode(0)
    return f


cases = [("per_layer", per_layer)]
if not os.environ.get("SKIP_RUN"):
    cases += [("persist1", runs(1)), ("persist8", runs(8)), ("persist32", runs(L)),
              ("warpbal32", moded(1, runs(L)))]
for name, fn in cases:
    us = timed(fn)
    st.check_errors()
    res[name + "_us_per_layer"] = us / L
    res[name + "_GBs"] = att_bytes / (us * 1e-6) / 1e9


def steps(run_kernel, n=32):
    eng.run_kernel = run_kernel
    eng._graphs.clear()
    eng.capture_graphs()
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        eng.step()
    b_.record()
    torch.cuda.synchronize()
    st.check_errors()
    return a.elapsed_time(b_) / n


if not os.environ.get("SKIP_RUN"):
    res["step_ms_run"] = steps(True)
res["step_ms_per_layer"] = steps(False)
print(json.dumps(res))
