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


def _pairs(st, *a, **k):
    return KVStore.cluster_map_pairs(st, *a, **k)


def test_pair_map_covers_every_head_and_pads():
    """Partial steps (rows at their own rerank): the due (row, head) pairs get
    a cluster of S CTAs each, every other head one CTA; the map is padded with
    idle CTAs to the launch's fixed grid."""
    st = _store()
    scored = {(3, h) for h in range(8)} | {(b, 0) for b in range(4)}  # 11 pairs: 22 + 117 <= 148
    S, n_ctas = 2, 148
    m = _pairs(st, 16, scored, S, n_ctas).tolist()
    assert len(m) == n_ctas
    split = [e for e in m if e >= 0 and not e & (1 << 30)]
    alone = [e & ~(1 << 30) for e in m if e >= 0 and e & (1 << 30)]
    assert sorted(set(split)) == sorted(b * 8 + h for (b, h) in scored)
    assert all(split.count(e) == S for e in set(split))
    assert sorted(set(split) | set(alone)) == list(range(16 * 8))  # every head exactly somewhere
    assert not set(split) & set(alone)


def test_pair_map_demotes_when_the_grid_is_short():
    """More due pairs than the captured grid holds: the surplus heads attend
    (and score) alone — every head is still covered (a map never drops one)."""
    st = _store()
    scored = {(b, h) for b in range(4) for h in range(8)}  # 32 pairs x 2 + 96 others = 160 > 136
    m = _pairs(st, 16, scored, 2, 136).tolist()
    assert len(m) == 136
    heads = {e & ~(1 << 30) for e in m if e >= 0}
    assert heads == set(range(16 * 8))


def test_cluster_plan_prefers_power_of_two_and_charges_the_select():
    st = _store(uniform_split=1)
    plan = KVStore.cluster_plan(st, 16, 8, 2049, 128, bw_sm_gbs=45.0, select_us=7.0)
    assert plan is not None and plan[0] in (2, 4, 8, 16) and plan[1] <= 148
    assert KVStore.cluster_plan(st, 16, 0, 2049, 128) is None        # nothing scored
    assert KVStore.cluster_plan(st, 16, 128, 2049, 128) is None      # everything scored
