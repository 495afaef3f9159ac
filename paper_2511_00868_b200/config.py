"""Hot-path configuration and head addressing.

Mirrors the fields of the reference ``Config`` (tierkv/config.py:27-108)
that the per-decode-step path reads, plus the GQA group size the reference
does not model.  Simulator cost-model fields are out of scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterator, NamedTuple

from .errors import ConfigError


class HeadId(NamedTuple):
    """(layer, head) address of one KV head (config.py:19-24)."""

    layer: int
    head: int


@dataclass(frozen=True)
class Config:
    page_size_tokens: int = 16      # config.py:30
    topk_pages: int = 64            # config.py:31
    unstable_fraction: float = 0.25  # config.py:32
    rerank_period: int = 16         # config.py:33
    stability_window: int = 32      # config.py:34 (head profiling window, decode steps)
    window_stride: int = 0          # config.py:35 (0 = non-overlapping windows)
    num_layers: int = 4             # config.py:37
    kv_heads_per_layer: int = 8     # config.py:38
    head_dim: int = 64              # config.py:39
    bytes_per_kv_element: int = 2   # config.py:40
    rng_seed: int = 12345           # config.py:48
    group_size: int = 1             # query heads per KV head (GQA; not in the reference)

    def __post_init__(self):
        for name in ("page_size_tokens", "topk_pages", "rerank_period", "num_layers",
                     "kv_heads_per_layer", "head_dim", "bytes_per_kv_element", "group_size",
                     "stability_window"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 1:
                raise ConfigError(f"{name} must be a positive integer, got {v!r}")
        if not 0.0 < self.unstable_fraction < 1.0:
            raise ConfigError(f"unstable_fraction must lie in (0, 1), got {self.unstable_fraction!r}")
        if self.stability_window < 2:
            raise ConfigError(f"stability_window must be >= 2, got {self.stability_window!r}")
        if not isinstance(self.window_stride, int) or self.window_stride < 0:
            raise ConfigError(f"window_stride must be a non-negative integer, got {self.window_stride!r}")
        if self.bytes_per_kv_element not in (2, 4):
            raise ConfigError("bytes_per_kv_element must be 2 (bf16) or 4 (fp32)")

    @property
    def stride(self) -> int:
        """Window stride; 0 means non-overlapping (config.py:92-93)."""
        return self.window_stride if self.window_stride else self.stability_window

    @property
    def n_heads(self) -> int:
        return self.num_layers * self.kv_heads_per_layer

    @property
    def page_bytes(self) -> int:
        """K and V bytes of one page of one head (config.py:95-98)."""
        return self.page_size_tokens * self.head_dim * 2 * self.bytes_per_kv_element

    @property
    def minmax_bytes_per_page(self) -> int:
        """config.py:100-103."""
        return 2 * self.head_dim * self.bytes_per_kv_element

    def n_unstable_heads(self, fraction: float | None = None) -> int:
        """round(fraction * L * H), half away from zero (config.py:105-108)."""
        f = self.unstable_fraction if fraction is None else fraction
        return int(math.floor(f * self.n_heads + 0.5))


def all_heads(cfg: Config) -> Iterator[HeadId]:
    for layer in range(cfg.num_layers):
        for head in range(cfg.kv_heads_per_layer):
            yield HeadId(layer, head)


def pages_for_tokens(tokens: int, page_size_tokens: int) -> int:
    """config.py:117-118."""
    return -(-tokens // page_size_tokens)


def full_pages_for_tokens(tokens: int, page_size_tokens: int) -> int:
    return tokens // page_size_tokens
