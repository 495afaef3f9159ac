"""Where a two-tier rerank step's time goes at config 3 (profiling aid):
wraps the engine's store calls with CUDA events during one eager rerank step
and prints per-call-kind device time (us) and counts."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402
from paper_2511_00868_b200.synthetic import device_normal  # noqa: E402

L, H, G, D, T, K, R, B = 32, 8, 4, 128, 32768, 128, 8, 1
dev = torch.device("cuda", 0)
prof = HeadProfile.first_n(L, H, 0.25)
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T + 200, topk_pages=K,
                   rerank_period=R, profile=prof, tiering=True, device=dev)
for l in range(L):
    eng.prefill_layer(0, l, device_normal((H, T, D), seed=2 * l), device_normal((H, T, D), seed=2 * l + 1),
                      alloc=(l == 0))
gen = torch.Generator(device=dev)
gen.manual_seed(1)
q = torch.randn(tuple(eng.q.shape), generator=gen, device=dev)


def feed():
    global q
    q = 0.99 * q + (1 - 0.99 ** 2) ** 0.5 * torch.randn(tuple(q.shape), generator=gen, device=dev)
    eng.q.copy_(q)
    eng.k_new.normal_(generator=gen)
    eng.v_new.normal_(generator=gen)


feed()
eng.step()
while not eng.is_rerank_step(eng.t + 1):
    feed()
    eng.step()
feed()
eng.step()  # the step before the rerank (staging in flight)
torch.cuda.synchronize()
times = collections.defaultdict(float)
counts = collections.Counter()
st = eng.store
targets = [(st, "score_select"), (st, "score_attend"), (st, "rerank_recycle"), (st, "sparse_decode"), (st, "sparse_decode_layers"),
           (st, "step_advance"), (st, "offload_filled"), (eng.stager, "fetch"), (eng.stager, "finish_rerank")]
pending = []
for obj, name in targets:
    fn = getattr(obj, name)

    def wrapped(*a, __fn=fn, __name=name, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = __fn(*a, **k)
        e1.record()
        pending.append((__name, e0, e1))
        return r
    setattr(obj, name, wrapped)
feed()
eng.stager.wait()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
eng._launch_step("rerank", force_due=False, fetch=eng._fetch_mode())
b.record()
torch.cuda.synchronize()
for name, e0, e1 in pending:
    times[name] += e0.elapsed_time(e1) * 1e3
    counts[name] += 1
print(json.dumps({"step_us_eager": a.elapsed_time(b) * 1e3,
                  "by_call_us": {k: round(v, 1) for k, v in times.items()}, "counts": dict(counts),
                  "copies_per_layer": eng.n_copies.tolist()}))
