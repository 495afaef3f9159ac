"""Post-prefill offload bandwidth (HBM pool -> pinned host) against the CTAs
the copy may occupy, alone and beside a decode step stream (serving)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_00868_b200.store import KVStore, PAGE_SIZE  # noqa: E402

B, L, H, D = 1, 8, 8, 128
T = 16384
pages = T // PAGE_SIZE
st = KVStore(batch_cap=B, layers=L, kv_heads=H, group=4, head_dim=D, pages_cap=pages + 1,
             n_blocks=B * L * H * (pages + 1) + 1, sel_cap=64, dtype=torch.bfloat16, device="cuda")
st.alloc_pages(0, 0, pages + 1)
host = torch.empty((B, L, H, pages + 1, 2, PAGE_SIZE, D), dtype=torch.bfloat16, pin_memory=True)
ent = torch.stack(torch.meshgrid(torch.zeros(1, dtype=torch.int32), torch.arange(L, dtype=torch.int32),
                                 torch.arange(H, dtype=torch.int32), torch.arange(pages, dtype=torch.int32),
                                 indexing="ij"), -1).reshape(-1, 4).cuda()
nbytes = ent.shape[0] * st.page_bytes
res = {"bytes": nbytes}
for ctas in (4, 8, 16, 24, 32, 64, 148, 0):
    st.offload_pages(host, ent, ctas)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        st.offload_pages(host, ent, ctas)
    b.record()
    b.synchronize()
    res[f"ctas_{ctas}_GBps"] = round(3 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9, 2)
# the copy engine for comparison: one contiguous D2H of the same bytes
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    dst.copy_(src, non_blocking=True)
b.record()
b.synchronize()
res["copy_engine_GBps"] = round(3 * nbytes / (a.elapsed_time(b) / 1e3) / 1e9, 2)
print(json.dumps(res))
