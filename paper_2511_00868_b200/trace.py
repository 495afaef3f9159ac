"""Top-K selection traces: the reference's FXTK container
(tierkv/trace.py:1-19) plus device-side capture from the decode engine.

* ``TopKTrace`` / ``save_trace`` / ``load_trace`` — the same container, the
  same invariants (trace.py:71-93) and the same ``TraceFormatError`` messages
  and byte offsets (trace.py:114-151), so traces move freely between the
  reference's tooling and this package.
* ``TraceRecorder`` — attaches to a ``DecodeEngine``: every step scores every
  head (a profiling step) and ``fc_trace_capture`` copies each head's top-K
  selection into an HBM trace buffer inside the step graph; one D2H copy at
  the end yields one ``TopKTrace`` per request row.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import HeadId
from .errors import TraceFormatError

MAGIC = b"FXTK"
VERSION = 1
_HEADER = struct.Struct("<4sIIHHH")  # magic, version, D, L, H, K


def _violation(sel: np.ndarray, pools: np.ndarray):
    """(message, step, record) of the first broken invariant, or None; record
    is the flat (l*H + h)*K + j position, or -1 for the pool field.  Order as
    the reference: pool shrink, index >= pool, duplicate within a record."""
    if sel.shape[0] == 0:
        return None
    d, L, H, K = sel.shape
    shrink = np.flatnonzero(np.diff(pools.astype(np.int64)) < 0)
    if shrink.size:
        s = int(shrink[0]) + 1
        return f"candidate pool shrinks at step {s} ({int(pools[s - 1])} -> {int(pools[s])})", s, -1
    over = sel >= pools.reshape(-1, 1, 1, 1)
    if over.any():
        s, l, h, j = (int(x) for x in np.unravel_index(int(np.argmax(over)), over.shape))
        return (f"page index {int(sel[s, l, h, j])} >= pool size {int(pools[s])} "
                f"at step {s}, layer {l}, head {h}", s, (l * H + h) * K + j)
    if K > 1:
        srt = np.sort(sel, axis=3)
        dup = (srt[..., 1:] == srt[..., :-1]).any(axis=3)
        if dup.any():
            s, l, h = (int(x) for x in np.unravel_index(int(np.argmax(dup)), dup.shape))
            return f"duplicate page index within selection at step {s}, layer {l}, head {h}", s, (l * H + h) * K
    return None


@dataclass
class TopKTrace:
    """Per-step top-K selections of every (layer, head) of one request
    (trace.py:36-70): selections (D, L, H, K) u32, pool_sizes (D,) u32."""

    sample_id: str
    selections: np.ndarray = field(repr=False)
    pool_sizes: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.selections = np.ascontiguousarray(self.selections, dtype=np.uint32)
        self.pool_sizes = np.ascontiguousarray(self.pool_sizes, dtype=np.uint32)
        if self.selections.ndim != 4:
            raise ValueError("selections must have shape (D, L, H, K)")
        if self.pool_sizes.shape != (self.selections.shape[0],):
            raise ValueError("pool_sizes must have one entry per step")
        bad = _violation(self.selections, self.pool_sizes)
        if bad is not None:
            raise ValueError(bad[0])

    @property
    def n_steps(self) -> int:
        return self.selections.shape[0]

    @property
    def n_layers(self) -> int:
        return self.selections.shape[1]

    @property
    def n_heads_per_layer(self) -> int:
        return self.selections.shape[2]

    @property
    def k(self) -> int:
        return self.selections.shape[3]

    def head_selections(self, head: HeadId) -> np.ndarray:
        return self.selections[:, head.layer, head.head, :]


def _pack(trace: TopKTrace) -> bytes:
    d, l, h, k = trace.selections.shape
    body = np.empty((d, 1 + l * h * k), dtype="<u4")
    body[:, 0] = trace.pool_sizes
    body[:, 1:] = trace.selections.reshape(d, -1)
    return _HEADER.pack(MAGIC, VERSION, d, l, h, k) + body.tobytes()


def save_trace(trace: TopKTrace, path) -> None:
    with open(path, "wb") as fh:
        fh.write(_pack(trace))


def parse_trace(blob: bytes, sample_id: str) -> TopKTrace:
    if len(blob) < _HEADER.size:
        raise TraceFormatError(f"truncated header: need {_HEADER.size} bytes, have {len(blob)}", 0)
    magic, version, d, l, h, k = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise TraceFormatError(f"bad magic {magic!r}, expected {MAGIC!r}", 0)
    if version != VERSION:
        raise TraceFormatError(f"unsupported version {version}", 4)
    if l == 0 or h == 0 or k == 0:
        raise TraceFormatError(f"zero dimension in header (L={l}, H={h}, K={k})", 12)
    rec = 1 + l * h * k  # u32 words per step
    want = _HEADER.size + d * rec * 4
    if len(blob) < want:
        raise TraceFormatError(f"truncated: need {want} bytes for {d} steps, have {len(blob)}", len(blob))
    if len(blob) > want:
        raise TraceFormatError("trailing data after last step", want)
    body = np.frombuffer(blob, dtype="<u4", count=d * rec, offset=_HEADER.size).reshape(d, rec)
    pools = body[:, 0].astype(np.uint32)
    sel = body[:, 1:].astype(np.uint32).reshape(d, l, h, k)
    bad = _violation(sel, pools)
    if bad is not None:
        msg, s, r = bad
        base = _HEADER.size + s * rec * 4
        raise TraceFormatError(msg, base if r < 0 else base + 4 + 4 * r)
    return TopKTrace(sample_id=sample_id, selections=sel, pool_sizes=pools)


def load_trace(path, sample_id: str | None = None) -> TopKTrace:
    with open(path, "rb") as fh:
        blob = fh.read()
    if sample_id is None:
        name = os.path.basename(str(path).replace("\\", "/"))
        sample_id = name.rsplit(".", 1)[0] if "." in name else name
    return parse_trace(blob, sample_id)


class TraceRecorder:
    """Capture top-K traces of a ``DecodeEngine`` run on the device.

    While attached, every engine step scores every head (a profiling step:
    the reference's traces record each head's selection at every step) and
    appends one FXTK step per request row to an HBM buffer
    [B, n_steps, L, H, K] u32 — inside the step graph, no host sync.
    ``traces()`` copies it back once and returns one ``TopKTrace`` per row.
    """

    def __init__(self, engine, n_steps: int, sample_ids=None):
        if n_steps < 1:
            raise ValueError("n_steps must be >= 1")
        self.eng = engine
        st = engine.store
        self.n_slots = n_steps
        self.sel = torch.zeros((engine.B, n_steps, engine.L, engine.H, engine.K), dtype=torch.int32,
                               device=st.device)
        self.pool = torch.zeros((engine.B, n_steps), dtype=torch.int32, device=st.device)
        self.t0 = engine.t
        self.step_base = engine.t + 1  # the device step after the first recorded advance
        self.sample_ids = list(sample_ids) if sample_ids is not None else [f"row{b}" for b in range(engine.B)]
        engine.attach_recorder(self)

    def capture(self) -> None:
        """Launched by the engine after the step advance (graph-capturable)."""
        e = self.eng
        e.store.trace_capture(self.sel, self.pool, self.step_base, e.K, e.B, extra_tokens=0)

    @property
    def n_recorded(self) -> int:
        return max(0, min(self.n_slots, self.eng.t - self.t0))

    def traces(self) -> list[TopKTrace]:
        self.eng.store.check_errors()
        n = self.n_recorded
        sel = self.sel[:, :n].cpu().numpy().view(np.uint32)
        pool = self.pool[:, :n].cpu().numpy().view(np.uint32)
        return [TopKTrace(self.sample_ids[b], sel[b], pool[b]) for b in range(self.eng.B)]
