import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2511_00868_b200.engine import DecodeEngine
from paper_2511_00868_b200.stability import HeadProfile
from paper_2511_00868_b200.config import HeadId
L,H,G,D,B,T,K,R=32,8,4,128,8,131072,128,16
prof = HeadProfile(model_id="x", n_layers=L, n_heads_per_layer=H, fraction=0.25, unstable=tuple(HeadId(l,h) for l in range(L) for h in range(2)))
eng = DecodeEngine(batch=B, layers=L, kv_heads=H, group=G, head_dim=D, ctx_cap_tokens=T+400, topk_pages=K, rerank_period=R, profile=prof)
for b in range(B): eng.seq_host[b] = T
print("supported", eng.store.score_attend_supported(B), "bal", eng.store.score_attend_balanced_supported(B))
print("use_balanced", eng._use_balanced(0, "plain", False))
p = eng._mixed_plan(0)
print("mixed plan", None if p is None else (p[1], p[0].numel()))
print("use_run", eng._use_run(), "run_split", eng.store.run_split(B, eng.att_bound))
