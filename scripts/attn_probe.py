"""Profiling probe: config-2 layer attention with a per-CTA timeline and a
sweep of grid sizes.  Prints a JSON summary (not a bench number)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_00868_b200.engine import DecodeEngine
from paper_2511_00868_b200.stability import HeadProfile
from paper_2511_00868_b200.synthetic import device_normal

B, L, H, G, D, T, K, R = 16, int(os.environ.get("L", 4)), 8, 4, 128, 32768, 128, 16
dev = torch.device("cuda", 0)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 64,
                   topk_pages=K, rerank_period=R, profile=HeadProfile.first_n(L, H, 0.25), device=dev)
srcs = [(device_normal((H, T, D), seed=2 * i), device_normal((H, T, D), seed=2 * i + 1)) for i in range(2)]
for b in range(B):
    for l in range(L):
        k, v = srcs[(b + l) % 2]
        eng.prefill_layer(b, l, k, v, alloc=(l == 0))
eng.q.copy_(device_normal(tuple(eng.q.shape), seed=99))
eng.step()  # initial selection
torch.cuda.synchronize()
st = eng.store
lib = st.lib
lib.fc_debug_attn_trace.restype = ctypes.c_int
lib.fc_debug_attn_trace.argtypes = [ctypes.c_void_p]
res = {}
alg = eng.attention_bytes(0)
for n_ctas in [0, 1, 2, 4]:
    ts = []
    for rep in range(5):
        for l in range(L):
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(5_000_000)
            a.record(); st.sparse_decode(l, eng.q[l], eng.out[l], B, max_pages=eng.att_bound, n_ctas=n_ctas, attend_appended=False); b_.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b_) * 1e3)
    ts.sort()
    res[n_ctas] = {"us_med": ts[len(ts) // 2], "us_min": ts[0], "GBs": alg / (ts[len(ts)//2] * 1e-6) / 1e9}
print(json.dumps(res))
# timeline at the default grid
grid = 2 * 148
buf = torch.zeros(8192 * 4, dtype=torch.int64, device=dev)
lib.fc_debug_attn_trace(buf.data_ptr())
torch.cuda._sleep(5_000_000)
st.sparse_decode(0, eng.q[0], eng.out[0], B, max_pages=eng.att_bound, attend_appended=False)
torch.cuda.synchronize()
lib.fc_debug_attn_trace(None)
tr = buf.view(-1, 4).cpu().numpy().astype("float64")
tr = tr[tr[:, 3] > 0]
t0 = tr[:, 0].min()
import numpy as np
def pct(x): return [round(float(np.percentile(x, p)), 2) for p in (0, 10, 50, 90, 100)] if len(x) else []
print(json.dumps({"ctas": int(tr.shape[0]), "entry": pct((tr[:, 0] - t0) / 1e3), "issued": pct((tr[:, 1] - t0) / 1e3),
                  "loop_done": pct((tr[:, 2] - t0) / 1e3), "exit": pct((tr[:, 3] - t0) / 1e3),
                  "body": pct((tr[:, 2] - tr[:, 1]) / 1e3), "merge": pct((tr[:, 3] - tr[:, 2]) / 1e3)}))

# ---- scoring: score only vs score + select (layer 0, all heads due)
def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(5_000_000)
        a.record(); fn(); b_.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b_) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]
sc_bytes = eng.scoring_bytes(0, 1)
t_sel = timeit(lambda: st.score_select(0, eng.q[0], eng.unstable, R, K, B, extra_tokens=1, force_due=True))
t_sc = timeit(lambda: st.score_pages(0, eng.q[0], B, extra_tokens=1))
t_att = timeit(lambda: st.sparse_decode(0, eng.q[0], eng.out[0], B, max_pages=eng.att_bound, attend_appended=False))
print(json.dumps({"score_select_us": t_sel, "score_only_us": t_sc, "attn_us": t_att,
                  "score_GBs": sc_bytes / (t_sc * 1e-6) / 1e9, "score_select_GBs": sc_bytes / (t_sel * 1e-6) / 1e9}))

lib.fc_debug_score_trace.restype = ctypes.c_int
lib.fc_debug_score_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(4096 * 4, dtype=torch.int64, device=dev)
lib.fc_debug_score_trace(buf.data_ptr())
torch.cuda._sleep(5_000_000)
st.score_select(0, eng.q[0], eng.unstable, R, K, B, extra_tokens=1, force_due=True)
torch.cuda.synchronize()
lib.fc_debug_score_trace(None)
tr = buf.view(-1, 4).cpu().numpy().astype("float64")
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
ent = (tr[:, 0] - t0) / 1e3
fin = (tr[:, 3] - t0) / 1e3
sc_done = (tr[:, 1] - t0) / 1e3
sel_rows = tr[:, 2] > 0
sel_start = sc_done[sel_rows]; sel_end = (tr[sel_rows, 2] - t0) / 1e3
print(json.dumps({"score_ctas": int(tr.shape[0]), "entry": pct(ent), "scoring_done": pct(sc_done), "exit": pct(fin),
                  "n_selectors": int(sel_rows.sum()), "select_us": pct(sel_end - sel_start), "select_end": pct(sel_end)}))

# ---- access-pattern probe: contiguous selections vs the top-K (scattered) ones
sel_bak, nsel_bak = st.sel.clone(), st.n_sel.clone()
n_att = int(st.n_sel[0, 0, 0].item())
contig = torch.arange(n_att, dtype=torch.int32, device=dev)
st.sel[:, 0, :, :n_att] = contig
t_contig = timeit(lambda: st.sparse_decode(0, eng.q[0], eng.out[0], B, max_pages=eng.att_bound, attend_appended=False))
st.sel.copy_(sel_bak); st.n_sel.copy_(nsel_bak)
t_sparse = timeit(lambda: st.sparse_decode(0, eng.q[0], eng.out[0], B, max_pages=eng.att_bound, attend_appended=False))
print(json.dumps({"attn_contiguous_pages_us": t_contig, "attn_topk_pages_us": t_sparse, "n_att": n_att}))
