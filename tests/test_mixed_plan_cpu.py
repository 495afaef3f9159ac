"""Host-side planning of mixed-cluster fused launches
(KVStore.mixed_cluster_map) with the device queries stubbed: no GPU."""

import types

import torch

from paper_2511_00868_b200.store import KVStore


def _store(H=8, D=128, uniform_split=2, fits=lambda n, s: True):
    st = types.SimpleNamespace(H=H, D=D, device=torch.device("cpu"),
                               kv_pool=torch.zeros(1, dtype=torch.bfloat16), _sms=148)
    st.page_bytes = 2 * 16 * D * 2
    st.score_attend_supported = lambda batch: uniform_split
    st.score_attend_map_fits = fits
    return st


def _plan(st, *a, **k):
    return KVStore.mixed_cluster_map(st, *a, **k)


def test_plan_covers_every_head_once():
    st = _store()
    m, S = _plan(st, 8, [0, 1], 8192, 128)  # config 4's shape, 2 of 8 heads scored
    m = m.tolist()
    assert len(m) % S == 0 and len(m) <= 148
    split = [e for e in m if e >= 0 and not e & (1 << 30)]
    alone = [e & ~(1 << 30) for e in m if e >= 0 and e & (1 << 30)]
    assert sorted(set(split)) == sorted(b * 8 + h for b in range(8) for h in (0, 1))
    assert all(split.count(e) == S for e in set(split))
    assert sorted(alone) == sorted(b * 8 + h for b in range(8) for h in range(2, 8))
    assert all(m[i:i + S] == [m[i]] * S for i in range(0, len(split), S))  # a split head fills its cluster


def test_no_plan_when_nothing_to_balance():
    st = _store()
    assert _plan(st, 8, [], 8192, 128) is None                 # nothing scored
    assert _plan(st, 8, list(range(8)), 8192, 128) is None     # every head scored: the uniform launch
    assert _plan(st, 16, [0, 1], 2048, 128) is None            # config 2: no one-wave mixed grid
    assert _plan(_store(fits=lambda n, s: False), 8, [0, 1], 8192, 128) is None
    assert _plan(_store(uniform_split=0), 8, [0, 1], 8192, 128) is None  # fused launch unsupported


def test_short_context_keeps_uniform():
    # at 2k tokens a scored head carries little more than an unscored one
    st = _store()
    assert _plan(st, 8, [0, 1], 128, 128) is None
