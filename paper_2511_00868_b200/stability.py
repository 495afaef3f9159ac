"""Head stability classification mask — the part of the reference's
``tierkv.stability`` the per-step path consumes: ``HeadProfile``
(stability.py:170-260).  The offline profiling that produces it (RCO,
temporal stability, classify_heads) runs once per model and is out of scope
(SURVEY.md §2); profiles written by the reference load here unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import HeadId
from .errors import ConsistencyError


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
