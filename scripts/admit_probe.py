"""CPU time spent inside engine.admit (tiered) while an earlier offload runs."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2511_00868_b200.engine import DecodeEngine  # noqa: E402
from paper_2511_00868_b200.stability import HeadProfile  # noqa: E402

L, H, D, T = 32, 8, 128, 16384
eng = DecodeEngine(batch=4, layers=L, kv_heads=H, group=4, head_dim=D, ctx_cap_tokens=T + 64, topk_pages=64,
                   rerank_period=8, profile=HeadProfile.first_n(L, H, 0.25), tiering=True,
                   n_blocks=4 * L * H * (T // 16 + 8))
eng.start_serving()
k = torch.randn((L, H, T, D), device="cuda", dtype=torch.bfloat16)
for row in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.prefill(row, k, k)
    t1 = time.perf_counter()
    eng.admit.__func__  # noqa
    cur = torch.cuda.current_stream()
    if eng.offload_stream is None:
        eng.offload_stream = torch.cuda.Stream()
    eng.offload_stream.wait_stream(cur)
    with torch.cuda.stream(eng.offload_stream):
        t2 = time.perf_counter()
        eng.tier.offload_after_prefill(row, T // 16, eng.offload_ctas)
        t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"row {row}: prefill cpu {1e3*(t1-t0):.1f} ms, offload cpu {1e3*(t3-t2):.1f} ms, "
          f"offload device-done {1e3*(t4-t3):.1f} ms", flush=True)

import cProfile  # noqa: E402
import pstats  # noqa: E402

eng.retire(1)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
with torch.cuda.stream(eng.offload_stream):
    eng.tier.offload_after_prefill(1, T // 16, eng.offload_ctas)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
