"""Head stability (tierkv.stability): the classification mask the decode step
consumes (``HeadProfile``, stability.py:170-260) and the profiling that
produces it from top-K traces: random-corrected overlap,
windowed temporal stability, bottom-fraction counts and classification
(stability.py:24-169, 271-313).

The integer core — |anchor ∩ later| for every (layer, head, window, offset)
— runs on the GPU (``fc_trace_overlap``); the float64 RCO and mean
arithmetic runs on the host on exactly the reference's expressions, so
reports and profiles are bit-identical to the reference's.  Profiles written
by either side load in the other.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import Config, HeadId
from .errors import ConsistencyError, DegeneratePoolError


def _iter_heads(n_layers, n_heads_per_layer):
    for l in range(n_layers):
        for h in range(n_heads_per_layer):
            yield HeadId(l, h)


@dataclass
class HeadProfile:
    """Per-head stable/unstable classification (stability.py:170-198)."""

    model_id: str
    n_layers: int
    n_heads_per_layer: int
    fraction: float
    unstable: tuple
    mean_ts: np.ndarray = field(repr=False, default=None)
    bottom_counts: np.ndarray = field(repr=False, default=None)
    task: str = ""
    trace_ids: tuple = ()

    def __post_init__(self):
        self.unstable = tuple(sorted(HeadId(*h) for h in self.unstable))
        self._unstable_set = frozenset(self.unstable)
        shape = (self.n_layers, self.n_heads_per_layer)
        if self.mean_ts is None:
            self.mean_ts = np.ones(shape)
        if self.bottom_counts is None:
            self.bottom_counts = np.zeros(shape, dtype=np.int64)

    @classmethod
    def first_n(cls, n_layers: int, n_heads_per_layer: int, fraction: float,
                model_id: str = "synthetic") -> "HeadProfile":
        """First round(fraction*L*H) flat heads unstable — the reference
        fixture ``make_profile`` (pkg/tests/conftest.py:21-33) with
        ``n_unstable_heads`` rounding (config.py:105-108)."""
        n = int(math.floor(fraction * n_layers * n_heads_per_layer + 0.5))
        heads = list(_iter_heads(n_layers, n_heads_per_layer))
        return cls(model_id=model_id, n_layers=n_layers, n_heads_per_layer=n_heads_per_layer,
                   fraction=n / (n_layers * n_heads_per_layer), unstable=tuple(heads[:n]))

    @property
    def n_heads(self) -> int:
        return self.n_layers * self.n_heads_per_layer

    @property
    def stable(self) -> tuple:
        return tuple(h for h in _iter_heads(self.n_layers, self.n_heads_per_layer)
                     if h not in self._unstable_set)

    def is_unstable(self, head) -> bool:
        return HeadId(*head) in self._unstable_set

    def mask(self) -> np.ndarray:
        """uint8 [L, H], 1 = unstable."""
        m = np.zeros((self.n_layers, self.n_heads_per_layer), dtype=np.uint8)
        for l, h in self.unstable:
            m[l, h] = 1
        return m

    def mask_tensor(self, device) -> torch.Tensor:
        return torch.as_tensor(self.mask()).to(device)

    # -- text format (stability.py:200-260): identical, so profiles interoperate

    def save_text(self, path) -> None:
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("# tierkv head profile v1\n")
            fh.write(f"# model_id={self.model_id}\n")
            fh.write(f"# task={self.task}\n")
            fh.write(f"# traces={','.join(self.trace_ids)}\n")
            fh.write(f"# fraction={self.fraction!r}\n")
            fh.write(f"# layers={self.n_layers}\n")
            fh.write(f"# heads_per_layer={self.n_heads_per_layer}\n")
            fh.write("# columns: layer head mean_ts bottom_count class\n")
            for l in range(self.n_layers):
                for h in range(self.n_heads_per_layer):
                    cls = "unstable" if HeadId(l, h) in self._unstable_set else "stable"
                    fh.write(f"{l} {h} {self.mean_ts[l, h]:.9g} "
                             f"{int(self.bottom_counts[l, h])} {cls}\n")

    @classmethod
    def load_text(cls, path) -> "HeadProfile":
        meta: dict = {}
        rows = []
        with open(path, "r", encoding="utf-8") as fh:
            for raw in fh:
                line = raw.strip()
                if not line:
                    continue
                if line.startswith("#"):
                    body = line[1:].strip()
                    if "=" in body:
                        k, _, v = body.partition("=")
                        meta[k.strip()] = v.strip()
                    continue
                parts = line.split()
                if len(parts) != 5:
                    raise ConsistencyError(f"{path}: malformed profile row {line!r}")
                rows.append(parts)
        try:
            l_dim, h_dim = int(meta["layers"]), int(meta["heads_per_layer"])
            fraction = float(meta.get("fraction", "0.25"))
        except (KeyError, ValueError) as exc:
            raise ConsistencyError(f"{path}: missing or malformed profile header") from exc
        if len(rows) != l_dim * h_dim:
            raise ConsistencyError(f"{path}: expected {l_dim * h_dim} head rows, found {len(rows)}")
        mean_ts = np.zeros((l_dim, h_dim))
        counts = np.zeros((l_dim, h_dim), dtype=np.int64)
        unstable = []
        for l_s, h_s, ts_s, c_s, klass in rows:
            l, h = int(l_s), int(h_s)
            mean_ts[l, h] = float(ts_s)
            counts[l, h] = int(c_s)
            if klass == "unstable":
                unstable.append(HeadId(l, h))
            elif klass != "stable":
                raise ConsistencyError(f"{path}: unknown head class {klass!r}")
        traces = tuple(t for t in meta.get("traces", "").split(",") if t)
        return cls(model_id=meta.get("model_id", ""), n_layers=l_dim, n_heads_per_layer=h_dim,
                   fraction=fraction, unstable=tuple(unstable), mean_ts=mean_ts,
                   bottom_counts=counts, task=meta.get("task", ""), trace_ids=traces)


# -- overlap primitives ------------------------------------------------------------

def _rco_value(intersection, k, pool_size):
    """max(0, (|A∩B|/K - K/N) / (1 - K/N)) (stability.py:41-42); numpy-vectorised."""
    chance = k / pool_size
    return np.maximum(0.0, (intersection / k - chance) / (1.0 - chance))


def rco(set_a, set_b, k: int, pool_size: int) -> float:
    """Random-corrected overlap of two K-subsets of a pool (stability.py:24-38)."""
    sa = {int(x) for x in set_a}
    sb = {int(x) for x in set_b}
    if len(sa) != k or len(sb) != k:
        raise ValueError(f"both sets must have exactly k={k} distinct elements")
    if k >= pool_size:
        raise DegeneratePoolError(f"overlap correction undefined: k={k} >= pool size {pool_size}")
    if sa and (max(sa) >= pool_size or max(sb) >= pool_size or min(sa) < 0 or min(sb) < 0):
        raise ValueError("set elements must lie in [0, pool_size)")
    return float(_rco_value(len(sa & sb), k, pool_size))


def _device_trace(trace, device):
    sel = torch.from_numpy(np.ascontiguousarray(trace.selections).view(np.int32)).to(device)
    pool = torch.from_numpy(np.ascontiguousarray(trace.pool_sizes).view(np.int32)).to(device)
    return sel, pool


def window_pair_values(trace, starts, window: int, device=None) -> np.ndarray:
    """RCO between each window's anchor step and every later step of the
    window, for every head: (L, H, n_windows, window - 1) float64, NaN where
    the later step's pool is degenerate (N_t <= K) — stability.py:45-62.
    Intersections come from ``fc_trace_overlap`` on the GPU."""
    from . import _lib
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    starts = [int(s) for s in starts]
    L, H, K = trace.n_layers, trace.n_heads_per_layer, trace.k
    if window < 2:
        raise ValueError("window must be >= 2")
    for s0 in starts:
        if s0 < 0 or s0 + window - 1 >= trace.n_steps:
            raise ValueError(f"window [{s0}, {s0 + window}) exceeds trace length {trace.n_steps}")
    vals = np.empty((L, H, len(starts), window - 1))
    if not starts:
        return vals
    sel, pool = _device_trace(trace, device)
    st = torch.tensor(starts, dtype=torch.int32, device=device)
    inter = torch.empty((L, H, len(starts), window - 1), dtype=torch.int32, device=device)
    max_pool = int(trace.pool_sizes.max())
    lib = _lib.load()
    _lib.check(lib.fc_trace_overlap(sel.data_ptr(), pool.data_ptr(), trace.n_steps, L, H, K, st.data_ptr(),
                                    len(starts), window, max_pool, inter.data_ptr(),
                                    torch.cuda.current_stream(device).cuda_stream), "fc_trace_overlap")
    inter = inter.cpu().numpy()
    later = np.asarray(starts)[:, None] + np.arange(1, window)[None, :]  # (W, window-1)
    pools = trace.pool_sizes.astype(np.int64)[later]
    degenerate = inter < 0
    with np.errstate(divide="ignore", invalid="ignore"):
        v = _rco_value(inter.astype(np.float64), K, np.where(pools > K, pools, K + 1)[None, None])
    vals[...] = np.where(degenerate, np.nan, v)
    return vals


def temporal_stability(trace, head: HeadId, start: int, window: int) -> float:
    """Mean anchored overlap of one head over one window; degenerate pairs
    are excluded (stability.py:65-76)."""
    if window < 2:
        raise ValueError("window must be >= 2")
    if start < 0 or start + window - 1 >= trace.n_steps:
        raise ValueError(f"window [{start}, {start + window}) exceeds trace length {trace.n_steps}")
    vals = window_pair_values(trace, [start], window)[head.layer, head.head, 0]
    good = vals[~np.isnan(vals)]
    if good.size == 0:
        raise DegeneratePoolError("every pair in the window has a degenerate pool")
    return float(good.sum() / good.size)


def _bottom_heads(ts_flat: np.ndarray, n_bottom: int) -> np.ndarray:
    """The n_bottom lowest-TS heads; ties toward the lower flat index (stability.py:131-137)."""
    return np.lexsort((np.arange(ts_flat.size), ts_flat))[:n_bottom]


@dataclass
class StabilityReport:
    """Windowed stability of one trace (stability.py:79-128)."""

    trace_id: str
    n_layers: int
    n_heads_per_layer: int
    window: int
    k: int
    window_starts: tuple
    ts: np.ndarray = field(repr=False)          # (L, H, n_windows)
    offset_rco: np.ndarray = field(repr=False)  # (L, H, window - 1)
    degenerate_pairs: int = 0

    @property
    def n_windows(self) -> int:
        return len(self.window_starts)

    @property
    def mean_ts(self) -> np.ndarray:
        return self.ts.mean(axis=2)

    def bottom_counts(self, fraction: float = 0.25) -> np.ndarray:
        n_bottom = int(math.floor(fraction * self.ts.shape[0] * self.ts.shape[1] + 0.5))
        counts = np.zeros(self.ts.shape[0] * self.ts.shape[1], dtype=np.int64)
        for w in range(self.ts.shape[2]):
            counts[_bottom_heads(self.ts[:, :, w].reshape(-1), n_bottom)] += 1
        return counts.reshape(self.ts.shape[:2])

    def save_text(self, path) -> None:
        mean, counts = self.mean_ts, self.bottom_counts()
        lines = ["# tierkv stability report v1", f"# trace={self.trace_id}", f"# layers={self.n_layers}",
                 f"# heads_per_layer={self.n_heads_per_layer}", f"# window={self.window}", f"# k={self.k}",
                 f"# windows={self.n_windows}", f"# degenerate_pairs={self.degenerate_pairs}",
                 "# columns: layer head mean_ts bottom_quartile_count"]
        lines += [f"{l} {h} {mean[l, h]:.9g} {int(counts[l, h])}"
                  for l in range(self.n_layers) for h in range(self.n_heads_per_layer)]
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("\n".join(lines) + "\n")


def compute_stability_report(trace, cfg: Config | None = None, *, window: int | None = None,
                             stride: int | None = None) -> StabilityReport:
    """Per-head temporal stability over windows of the trace (stability.py:140-169)."""
    if window is None:
        window = cfg.stability_window if cfg is not None else 32
    if stride is None:
        stride = cfg.stride if cfg is not None else window
    if window < 2:
        raise ValueError("window must be >= 2")
    if stride < 1:
        raise ValueError("stride must be >= 1")
    if trace.n_steps < window:
        raise ValueError(f"trace has {trace.n_steps} steps, too short for window {window}")
    starts = tuple(range(0, trace.n_steps - window + 1, stride))
    vals = window_pair_values(trace, starts, window)
    degenerate = int(np.isnan(vals).sum())
    with np.errstate(invalid="ignore"):
        ts = np.nanmean(vals, axis=3)
        offset_rco = np.nanmean(vals, axis=2)
    if np.isnan(ts).any():
        raise DegeneratePoolError("a window has no non-degenerate pairs")
    return StabilityReport(trace_id=trace.sample_id, n_layers=trace.n_layers,
                           n_heads_per_layer=trace.n_heads_per_layer, window=window, k=trace.k,
                           window_starts=starts, ts=ts, offset_rco=offset_rco, degenerate_pairs=degenerate)


def classify_heads(reports, fraction: float, *, model_id: str = "model", task: str = "") -> HeadProfile:
    """Mark the round(fraction*L*H) most frequently bottom-ranked heads
    unstable; ties toward lower mean TS, then lower flat index; invariant to
    report order (stability.py:271-313)."""
    reports = list(reports)
    if not reports:
        raise ValueError("classify_heads needs at least one report")
    if not 0.0 < fraction < 1.0:
        raise ValueError(f"fraction must lie in (0, 1), got {fraction!r}")
    L, H = reports[0].n_layers, reports[0].n_heads_per_layer
    if any((r.n_layers, r.n_heads_per_layer) != (L, H) for r in reports):
        raise ValueError("reports disagree on head grid dimensions")
    if sum(r.n_windows for r in reports) < 1:
        raise ValueError("no stability windows across the given reports")
    canon = sorted(reports, key=lambda r: (r.trace_id, r.n_windows, r.ts.tobytes()))
    n = L * H
    n_unstable = int(math.floor(fraction * n + 0.5))
    counts = np.zeros(n, dtype=np.int64)
    ts_sum = np.zeros(n)
    n_windows = 0
    for r in canon:
        for w in range(r.n_windows):
            counts[_bottom_heads(r.ts[:, :, w].reshape(-1), n_unstable)] += 1
        ts_sum += r.ts.sum(axis=2).reshape(-1)
        n_windows += r.n_windows
    mean_ts = ts_sum / n_windows
    order = np.lexsort((np.arange(n), mean_ts, -counts))  # (-count, mean TS, index)
    unstable = tuple(sorted(HeadId(int(i) // H, int(i) % H) for i in order[:n_unstable]))
    return HeadProfile(model_id=model_id, n_layers=L, n_heads_per_layer=H, fraction=fraction,
                       unstable=unstable, mean_ts=mean_ts.reshape(L, H),
                       bottom_counts=counts.reshape(L, H), task=task,
                       trace_ids=tuple(r.trace_id for r in canon))


def cross_task_overlap(profiles) -> np.ndarray:
    """Pairwise |A_i ∩ A_j| / C of the profiles' unstable sets (stability.py:316-338)."""
    profiles = list(profiles)
    if not profiles:
        raise ValueError("cross_task_overlap needs at least one profile")
    dims = (profiles[0].n_layers, profiles[0].n_heads_per_layer)
    card = len(profiles[0].unstable)
    if card == 0:
        raise ValueError("profiles have empty unstable sets")
    for p in profiles:
        if (p.n_layers, p.n_heads_per_layer) != dims:
            raise ValueError("profiles disagree on head grid dimensions")
        if len(p.unstable) != card:
            raise ValueError(f"unstable-set cardinality mismatch: {len(p.unstable)} != {card}")
    masks = np.stack([p.mask().reshape(-1).astype(np.int64) for p in profiles])
    out = (masks @ masks.T) / card
    np.fill_diagonal(out, 1.0)
    return out


def save_overlap_csv(matrix: np.ndarray, labels, path) -> None:
    """stability.py:341-349."""
    labels = list(labels)
    if matrix.shape != (len(labels), len(labels)):
        raise ValueError("label count must match matrix dimensions")
    rows = ["task," + ",".join(labels)]
    rows += [lab + "," + ",".join(f"{matrix[i, j]:.4f}" for j in range(len(labels)))
             for i, lab in enumerate(labels)]
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(rows) + "\n")
