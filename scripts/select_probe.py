import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_00868_b200.scoring import select_topk_device
res = {}
for heads in (1, 128):
    for n in (2047, 8191):
        sc = (torch.randn(heads, n, device="cuda") * 50 + 200).contiguous()
        nv = torch.full((heads,), n, dtype=torch.int32, device="cuda")
        out = torch.empty(heads, 128, dtype=torch.int32, device="cuda")
        no = torch.empty(heads, dtype=torch.int32, device="cuda")
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)
            a.record(); select_topk_device(sc, nv, 128, True, out, no); b.record()
            torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
        res[f"{heads}x{n}"] = sorted(ts)[2]
print(json.dumps(res))
