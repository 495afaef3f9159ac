"""Seeded synthetic inputs (the reference has no datasets or weights on
this path)."""

from __future__ import annotations

import numpy as np
import torch


def gen_synthetic_kv(cfg, tokens: int, seed: int | None = None):
    """Deterministic unit-scale key/value arrays of shape (L, H, tokens, d):
    keys then values drawn from ``np.random.default_rng(seed)`` — the draw
    order of the reference ``gen_synthetic_kv`` (trace.py:217-225), so a seed
    gives the reference's own float64 inputs."""
    if tokens < 0:
        raise ValueError("tokens must be non-negative")
    rng = np.random.default_rng(cfg.rng_seed if seed is None else seed)
    shape = (cfg.num_layers, cfg.kv_heads_per_layer, tokens, cfg.head_dim)
    return rng.standard_normal(shape), rng.standard_normal(shape)


def device_normal(shape, *, seed: int, dtype=torch.bfloat16, device="cuda") -> torch.Tensor:
    """N(0,1) tensor generated on the GPU (bench-scale inputs; 64 GiB of KV
    is not generated on the host)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn(shape, generator=g, dtype=torch.float32, device=device).to(dtype)


def ar1_queries(prev: torch.Tensor, rho: float, *, generator: torch.Generator) -> torch.Tensor:
    """q_t = rho q_{t-1} + sqrt(1 - rho^2) eps (drifting
    stable-head queries so consecutive reranks overlap, Appendix A.4)."""
    eps = torch.randn(prev.shape, generator=generator, dtype=torch.float32, device=prev.device)
    return (rho * prev.float() + (1.0 - rho * rho) ** 0.5 * eps).to(prev.dtype)
