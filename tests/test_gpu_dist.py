"""The KV-head-sharded decode (config 5's layout, SURVEY.md §8e option (i)) run
as 2 ranks on ONE GPU: two processes, gloo over CUDA tensors (the same
HeadGroup.gather code path as NCCL up to the collective call), each rank
owning half of the KV heads of every layer and all-gathering the attention
outputs after each layer.  The gathered outputs of every step must equal the
1-rank engine's (all heads in one process, same inputs) bit for bit: a query
head's attention is entirely local to the rank owning its KV head, so
sharding moves no arithmetic.  (The gpurun pool and the driver's round-end
tests have one GPU; NCCL refuses two ranks on one device.)"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

L, H, G, D, B, T, K, R, STEPS = 2, 4, 7, 128, 2, 1100, 16, 4, 7


def _inputs():
    from oracle import flexicache_oracle as O
    rng = np.random.default_rng(21)
    kv = [O.bf16_round(rng.standard_normal((B, L, H, T, D))) for _ in range(2)]
    steps = [tuple(O.bf16_round(rng.standard_normal(s)) for s in ((L, B, H * G, D), (L, B, H, D), (L, B, H, D)))
             for _ in range(STEPS)]
    return kv, steps


def run_sharded(rank: int, world: int):
    """Outputs [STEPS][L, B, H*G, D] (float32 numpy) of the head-sharded
    engine on this rank (world 1: every head here)."""
    import ctypes
    from paper_2511_00868_b200 import _lib
    from paper_2511_00868_b200 import dist as fdist
    from paper_2511_00868_b200.engine import DecodeEngine
    from paper_2511_00868_b200.stability import HeadProfile
    # the automatic cluster splits depend on the heads per launch (a shard
    # has half): pin them so both layouts split each head alike
    _lib.load().fc_debug_max_cluster.argtypes = [ctypes.c_int]
    _lib.load().fc_debug_max_cluster(8)
    heads, rows, _ = fdist.head_shard_of(rank, world, H, B)
    Hl = len(heads)
    # u = 0.25 with the same per-layer pattern on every shard (heads 0 and 2
    # of layer 0), so each rank launches the kernels the 1-rank engine does
    # (a shard's launch choice depends only on its own heads)
    unstable = ((0, 0), (0, 2))
    prof = HeadProfile(model_id="x", n_layers=L, n_heads_per_layer=Hl, fraction=0.25,
                       unstable=tuple((l, h - heads.start) for (l, h) in unstable if h in heads))
    group = fdist.HeadGroup(world, H)
    dev = torch.device("cuda", 0)
    out_full = torch.zeros((L, B, H * G, D), dtype=torch.bfloat16, device=dev)
    holder = {}

    def gather(layer):
        group.gather(holder["eng"].out[layer], out_full[layer])

    eng = DecodeEngine(batch=B, layers=L, kv_heads=Hl, group=G, head_dim=D, ctx_cap_tokens=T + STEPS + 32,
                       topk_pages=K, rerank_period=R, profile=prof, after_layer=gather)
    eng.mixed_clusters = False  # (maps are sized per launch: a shard's would differ from the whole)
    holder["eng"] = eng
    (k0, v0), steps = _inputs()
    hs = slice(heads.start, heads.stop)
    qs = slice(heads.start * G, heads.stop * G)
    for b in range(B):
        eng.prefill(b, torch.as_tensor(k0[b][:, hs]).to(dev).bfloat16(), torch.as_tensor(v0[b][:, hs]).to(dev).bfloat16())
    outs = []
    for q, kn, vn in steps:
        eng.q.copy_(torch.as_tensor(q[:, :, qs]))
        eng.k_new.copy_(torch.as_tensor(kn[:, :, hs]))
        eng.v_new.copy_(torch.as_tensor(vn[:, :, hs]))
        eng.step(use_graph=False)  # (a gloo collective cannot be captured in a CUDA graph)
        torch.cuda.synchronize()
        eng.store.check_errors()
        outs.append(out_full.float().cpu().numpy())
    _lib.load().fc_debug_max_cluster(0)
    return outs


def _rank_main(rank, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2511_00868_b200 import dist as fdist
    try:
        r, w, _ = fdist.init(backend="gloo")
        outs = run_sharded(r, w)
        if r == 0:
            q.put(("ok", outs))
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put(("err", f"rank {rank}: {e!r}"))
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_head_sharded_two_ranks_equal_one_rank_bitwise():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    assert all(p.exitcode == 0 for p in procs)
    ref = run_sharded(0, 1)
    assert len(payload) == len(ref) == STEPS
    for s, (got, want) in enumerate(zip(payload, ref)):
        assert np.isfinite(got).all()
        bad = np.argwhere((got != want).any(-1))  # (layer, row, query head)
        assert np.array_equal(got, want), (s, float(np.abs(got - want).max()), bad[:8].tolist())
