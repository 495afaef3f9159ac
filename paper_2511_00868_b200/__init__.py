"""B200-native FlexiCache per-decode-step KV hot path (sm_100a).

Drop-in for the hot-path API of the reference package ``tierkv``
(/root/reference/pkg/src/tierkv/__init__.py:22-54): head stability mask,
page table, score / select / attend / rerank calls.  All numerics run in the
hand-written CUDA library ``libflexicache_b200.so`` behind the C ABI in
include/flexicache_b200.h; PyTorch provides device memory and streams.
"""

from .config import Config, HeadId, all_heads, pages_for_tokens
from .errors import (AdmissionError, ConfigError, ConsistencyError, DegeneratePoolError,
                     PoolExhausted, TierKVError, TraceFormatError)

__version__ = "0.1.0"

_LAZY = {
    "KVStore": ".store", "DecodeEngine": ".engine", "HeadProfile": ".stability",
    "MinMaxMeta": ".scoring", "MinMaxCache": ".scoring", "TopKSet": ".scoring",
    "build_minmax": ".scoring", "update_minmax": ".scoring", "score_pages": ".scoring",
    "score_page": ".scoring", "select_topk": ".scoring", "rerank_due": ".scoring",
    "layer_scoring_skippable": ".scoring", "AttentionState": ".attention",
    "dense_decode": ".attention", "sparse_decode": ".attention",
    "sparsity_error": ".attention", "BlockTable": ".blocktable",
    "PhysicalPool": ".blocktable", "RecyclePlan": ".blocktable", "NULL_BLOCK": ".blocktable",
    "promoted_delta": ".tiering", "TierStore": ".tiering",
    "TopKTrace": ".trace", "save_trace": ".trace", "load_trace": ".trace",
    "TraceRecorder": ".trace", "rco": ".stability", "temporal_stability": ".stability",
    "StabilityReport": ".stability", "compute_stability_report": ".stability",
    "classify_heads": ".stability", "cross_task_overlap": ".stability",
    "save_overlap_csv": ".stability",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod = importlib.import_module(_LAZY[name], __name__)
        return getattr(mod, name)
    raise AttributeError(name)


__all__ = sorted(["Config", "HeadId", "all_heads", "pages_for_tokens", "AdmissionError",
                  "ConfigError", "ConsistencyError", "DegeneratePoolError", "PoolExhausted",
                  "TierKVError", "TraceFormatError", *_LAZY])
