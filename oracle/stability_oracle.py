"""CPU oracle for the selection-trace / head-stability row.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker, never by the
product path (paper_2511_00868_b200 computes intersections on the GPU and
fails loudly without its CUDA library).

A restatement of the reference's algorithms, each function citing the file
and lines it follows (pkg/src/tierkv/...):

* FXTK container (trace.py:1-19 format, :114-151 load validation order,
  :71-93 invariants) — ``fxtk_pack`` / ``fxtk_parse``;
* random-corrected overlap (stability.py:24-42), anchored window pair values
  (:45-62), the report (:140-169) and bottom-fraction counts (:98-107, 131-137);
* classification (stability.py:271-313);
* the synthetic planted-split generator (trace.py:160-209), restated with the
  same random-number call sequence so larger cases can be generated in-process.

Parity is pinned by tests/golden/trace_golden.json and the two .fxtk files,
written by the reference itself (tests/golden/make_golden_trace.py).
"""

from __future__ import annotations

import math
import struct

import numpy as np

MAGIC = b"FXTK"
HEADER = struct.Struct("<4sIIHHH")  # magic, version, D, L, H, K (18 bytes)


class FormatError(Exception):
    def __init__(self, message, offset):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


def first_violation(sel, pools):
    """(message, step, record) of the first broken invariant or None; record
    = l*H + h, or -1 for the pool field (trace.py:71-93: shrink, then index
    range, then duplicates)."""
    d = sel.shape[0]
    if d == 0:
        return None
    p = pools.astype(np.int64)
    for s in range(1, d):
        if p[s] < p[s - 1]:
            return (f"candidate pool shrinks at step {s} ({p[s - 1]} -> {p[s]})", s, -1)
    for s in range(d):
        bad = np.argwhere(sel[s] >= pools[s])
        if bad.size:
            l, h, j = map(int, bad[0])
            return (f"page index {int(sel[s, l, h, j])} >= pool size {int(pools[s])} "
                    f"at step {s}, layer {l}, head {h}", s, (l * sel.shape[2] + h) * sel.shape[3] + j)
    if sel.shape[3] > 1:
        for s in range(d):
            for l in range(sel.shape[1]):
                for h in range(sel.shape[2]):
                    if len(set(sel[s, l, h].tolist())) != sel.shape[3]:
                        return (f"duplicate page index within selection at step {s}, "
                                f"layer {l}, head {h}", s, (l * sel.shape[2] + h) * sel.shape[3])
    return None


def fxtk_pack(sel, pools) -> bytes:
    d, l, h, k = sel.shape
    parts = [HEADER.pack(MAGIC, 1, d, l, h, k)]
    for s in range(d):
        parts.append(struct.pack("<I", int(pools[s])))
        parts.append(np.asarray(sel[s], dtype="<u4").tobytes())
    return b"".join(parts)


def fxtk_parse(blob: bytes):
    """(sel (D,L,H,K) u32, pools (D,) u32) or FormatError with the reference's
    message and byte offset (trace.py:114-151)."""
    if len(blob) < HEADER.size:
        raise FormatError(f"truncated header: need {HEADER.size} bytes, have {len(blob)}", 0)
    magic, version, d, l, h, k = HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}", 0)
    if version != 1:
        raise FormatError(f"unsupported version {version}", 4)
    if l == 0 or h == 0 or k == 0:
        raise FormatError(f"zero dimension in header (L={l}, H={h}, K={k})", 12)
    step = 4 + l * h * k * 4
    want = HEADER.size + d * step
    if len(blob) < want:
        raise FormatError(f"truncated: need {want} bytes for {d} steps, have {len(blob)}", len(blob))
    if len(blob) > want:
        raise FormatError("trailing data after last step", want)
    pools = np.zeros(d, dtype=np.uint32)
    sel = np.zeros((d, l, h, k), dtype=np.uint32)
    for s in range(d):
        off = HEADER.size + s * step
        pools[s] = struct.unpack_from("<I", blob, off)[0]
        sel[s] = np.array(struct.unpack_from(f"<{l * h * k}I", blob, off + 4), dtype=np.uint32).reshape(l, h, k)
    bad = first_violation(sel, pools)
    if bad is not None:
        msg, s, rec = bad
        off = HEADER.size + s * step
        raise FormatError(msg, off if rec < 0 else off + 4 + 4 * rec)
    return sel, pools


# -- overlap and stability ------------------------------------------------------

def rco_value(inter: int, k: int, pool: int) -> float:
    """stability.py:41-42: max(0, (|A∩B|/K - K/N) / (1 - K/N))."""
    chance = k / pool
    return max(0.0, (inter / k - chance) / (1.0 - chance))


def pair_values(sel, pools, l, h, start, window):
    """stability.py:45-62: RCO(anchor, anchor+delta), NaN where N_t <= K."""
    k = sel.shape[3]
    anchor = set(sel[start, l, h].tolist())
    out = np.empty(window - 1)
    for delta in range(1, window):
        t = start + delta
        pool = int(pools[t])
        if k >= pool:
            out[delta - 1] = np.nan
            continue
        out[delta - 1] = rco_value(len(anchor & set(sel[t, l, h].tolist())), k, pool)
    return out


def report(sel, pools, window, stride):
    """stability.py:140-169 -> (starts, ts (L,H,W), offset_rco (L,H,window-1),
    degenerate count)."""
    d, L, H, _ = sel.shape
    starts = tuple(range(0, d - window + 1, stride))
    vals = np.empty((L, H, len(starts), window - 1))
    for l in range(L):
        for h in range(H):
            for w, s in enumerate(starts):
                vals[l, h, w] = pair_values(sel, pools, l, h, s, window)
    with np.errstate(invalid="ignore"):
        ts = np.nanmean(vals, axis=3)
        off = np.nanmean(vals, axis=2)
    return starts, ts, off, int(np.isnan(vals).sum())


def bottom_heads(ts_flat, n_bottom):
    """stability.py:131-137: lowest TS first, ties toward the lower flat index."""
    return np.lexsort((np.arange(ts_flat.size), ts_flat))[:n_bottom]


def bottom_counts(ts, fraction):
    """stability.py:98-107."""
    n = int(math.floor(fraction * ts.shape[0] * ts.shape[1] + 0.5))
    counts = np.zeros(ts.shape[0] * ts.shape[1], dtype=np.int64)
    for w in range(ts.shape[2]):
        counts[bottom_heads(ts[:, :, w].reshape(-1), n)] += 1
    return counts.reshape(ts.shape[:2])


def classify(reports, fraction):
    """stability.py:271-313 over [(trace_id, ts (L,H,W))]: canonical order,
    summed bottom counts and TS, rank by (-count, mean TS, flat index).
    Returns (unstable [(l,h)], counts (L,H), mean_ts (L,H), trace ids)."""
    L, H = reports[0][1].shape[:2]
    canon = sorted(reports, key=lambda r: (r[0], r[1].shape[2], r[1].tobytes()))
    n = L * H
    n_unstable = int(math.floor(fraction * n + 0.5))
    counts = np.zeros(n, dtype=np.int64)
    ts_sum = np.zeros(n)
    nw = 0
    for _, ts in canon:
        for w in range(ts.shape[2]):
            counts[bottom_heads(ts[:, :, w].reshape(-1), n_unstable)] += 1
        ts_sum += ts.sum(axis=2).reshape(-1)
        nw += ts.shape[2]
    mean = ts_sum / nw
    ranked = sorted(range(n), key=lambda i: (-counts[i], mean[i], i))
    unstable = sorted((i // H, i % H) for i in ranked[:n_unstable])
    return unstable, counts.reshape(L, H), mean.reshape(L, H), tuple(r[0] for r in canon)


def gen_planted_trace(L, H, K, page_size, planted, persistence, steps, initial_pool, seed):
    """trace.py:160-209 restated (same default_rng call sequence)."""
    unstable = np.zeros((L, H), dtype=bool)
    for l, h in planted:
        unstable[l, h] = True
    rng = np.random.default_rng(seed)
    sel = np.empty((steps, L, H, K), dtype=np.uint32)
    pools = np.empty(steps, dtype=np.uint32)
    for s in range(steps):
        pool = initial_pool + s // page_size
        pools[s] = pool
        for l in range(L):
            for h in range(H):
                if s == 0 or unstable[l, h]:
                    row = rng.choice(pool, size=K, replace=False)
                elif persistence >= 1.0:
                    row = sel[s - 1, l, h]
                else:
                    prev = sel[s - 1, l, h]
                    kept = prev[rng.random(K) < persistence]
                    need = K - kept.size
                    if need:
                        free = np.ones(pool, dtype=bool)
                        free[kept] = False
                        row = np.concatenate([kept, rng.choice(np.flatnonzero(free), size=need,
                                                               replace=False)])
                    else:
                        row = kept
                sel[s, l, h] = np.sort(row.astype(np.uint32))
    return sel, pools
