"""ctypes binding of the C ABI in include/flexicache_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
as ``paper_2511_00868_b200/libflexicache_b200.so``.  There is no fallback:
if the library is missing or no CUDA device is present, every product call
raises.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import CudaError, UnsupportedError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        os.environ.get("FC_LIB_VARIANT", "libflexicache_b200.so"))  # (A/B builds, profiling)
HEADER_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "include", "flexicache_b200.h")

FC_OK, FC_E_INVALID, FC_E_UNSUPPORTED, FC_E_CUDA, FC_E_CAPACITY = 0, -1, -2, -3, -4
FC_BF16, FC_F32 = 0, 1
FC_ERR_POOL_EXHAUSTED = 1
FC_ERR_NULL_READ = 2
FC_ERR_NULL_WRITE = 4
FC_ERR_PAGES_CAP = 8
FC_ERR_SEL_CAP = 16
FC_ERR_DOUBLE_EVICT = 32
FC_ERR_WRITE_TWICE = 64
FC_ERR_TRACE_SHORT = 128
FC_HOLD_NONE, FC_HOLD_WAIT, FC_HOLD_RESUME, FC_HOLD_RERANK = 0, 1, 2, 3
FC_STAT_SCORE_EVALS, FC_STAT_SCORE_EVALS_NAIVE, FC_STAT_LAYER_SKIPS, FC_STAT_HELD_ROW_STEPS = 0, 1, 2, 3
FC_STATS_N = 4

_p = ctypes.c_void_p
_i = ctypes.c_int
_f = ctypes.c_float
_i64 = ctypes.c_int64
_sz = ctypes.c_size_t


class FcStore(ctypes.Structure):
    """Mirror of ``struct fc_store`` (include/flexicache_b200.h)."""

    _fields_ = [
        ("batch_cap", ctypes.c_int32), ("layers", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32), ("group", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("page_size", ctypes.c_int32),
        ("pages_cap", ctypes.c_int32), ("sel_cap", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
        ("kv_pool", _p), ("summaries", _p), ("table", _p), ("seq_len", _p),
        ("sel", _p), ("n_sel", _p), ("free_stack", _p), ("free_top", _p),
        ("step", _p), ("error_word", _p),
        ("row_phase", _p), ("row_hold", _p), ("stats", _p),
    ]


_SIGNATURES = {
    "fc_version": (ctypes.c_char_p, []),
    "fc_last_error": (ctypes.c_char_p, []),
    "fc_alloc_pages": (_i, [_p, _i, _i, _i, _p]),
    "fc_free_row": (_i, [_p, _i, _p]),
    "fc_step_advance": (_i, [_p, _i, _p]),
    "fc_step_advance_counted": (_i, [_p, _i, _p, _i, _p]),
    "fc_select_topk_f64": (_i, [_p, _i, _i, _i, _p, _p, _p, _p]),
    "fc_kv_prefill": (_i, [_p, _i, _i, _p, _p, _i, _p]),
    "fc_kv_append": (_i, [_p, _i, _p, _p, _i, _p]),
    "fc_kv_gather": (_i, [_p, _i, _i, _i, _i, _p, _p, _p]),
    "fc_score_select_workspace_size": (_sz, [_p]),
    "fc_score_select": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p, _i, _p]),
    "fc_score_pages": (_i, [_p, _i, _p, _i, _p, _i, _p]),
    "fc_select_topk": (_i, [_p, _i, _p, _i, _i, _i, _p, _p, _p]),
    "fc_sparse_decode_workspace_size": (_sz, [_p, _i, _i, _i]),
    "fc_sparse_decode": (_i, [_p, _i, _p, _p, _p, _p, _p, _f, _i, _i, _i, _p, _i, _i, _i, _p, _sz, _i, _p]),
    "fc_score_attend_supported": (_i, [_p, _i]),
    "fc_score_attend": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _f, _i, _i, _p]),
    "fc_score_attend_map_fits": (_i, [_p, _i, _i]),
    "fc_score_attend_balanced_supported": (_i, [_p, _i]),
    "fc_score_attend_balanced": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _f, _i, _i, _p]),
    "fc_score_attend_balanced_workspace_size": (_sz, [_p, _i]),
    "fc_score_attend_balanced_ws": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _f, _i, _i, _p,
                                         _sz, _p]),
    "fc_score_attend_map": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _f, _i, _i, _p, _i, _i,
                                 _p]),
    "fc_sparse_decode_layers_supported": (_i, [_p, _i, _i]),
    "fc_sparse_decode_layers_split": (_i, [_p, _i, _i]),
    "fc_sparse_decode_layers_workspace_size": (_sz, [_p, _i, _i]),
    "fc_sparse_decode_layers": (_i, [_p, _i, _i, _p, _i64, _p, _p, _i64, _p, _i64, _p, _i64, _f, _i, _i, _i, _i,
                                     _p, _sz, _i, _p]),
    "fc_rerank_workspace_size": (_sz, [_p]),
    "fc_rerank_recycle": (_i, [_p, _i, _p, _p, _p, _i, _i, _i, _i, _p, _p, _i, _p, _p, _i, _p]),
    "fc_rerank_recycle_rows": (_i, [_p, _i, _p, _p, _p, _i, _i, _i, _i, _p, _p, _p, _i, _p, _p, _i, _p]),
    "fc_fetch_pages": (_i, [_p, _i, _p, _p, _p, _i, _p]),
    "fc_offload_pages": (_i, [_p, _p, _p, _i, _p]),
    "fc_offload_pages_ctas": (_i, [_p, _p, _p, _i, _i, _p]),
    "fc_fetch_pages_ctas": (_i, [_p, _i, _p, _p, _p, _i, _i, _i, _p]),
    "fc_fetch_pages_staged": (_i, [_p, _i, _p, _p, _p, _i, _p, _p, _p, _p]),
    "fc_stage_promoted": (_i, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _p, _i, _p]),
    "fc_stage_clear": (_i, [_p, _p, _p, _p, _i, _p]),
    "fc_stage_plan": (_i, [_p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _p]),
    "fc_stage_fetch": (_i, [_p, _p, _p, _p, _i, _p, _i, _p]),
    "fc_evict_pages": (_i, [_p, _p, _i, _p]),
    "fc_offload_filled": (_i, [_p, _p, _p, _p, _i, _p]),
    "fc_evict_unselected": (_i, [_p, _p, _i, _p]),
    "fc_trace_capture": (_i, [_p, _p, _p, _i, _i, _i, _i, _i, _p]),
    "fc_trace_overlap": (_i, [_p, _p, _i, _i, _i, _i, _p, _i, _i, _i, _p, _p]),
}

_lib = None


def header_symbols() -> list[str]:
    """Function names declared in include/flexicache_b200.h."""
    with open(HEADER_PATH) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fc_[a-z_0-9]+)\s*\(", text)))


def load():
    """Load the library (once) and attach prototypes; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback for the FlexiCache hot path")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI status to the reference's exception types."""
    capture_probe(what)
    if rc == FC_OK:
        return
    msg = load().fc_last_error().decode(errors="replace")
    if rc == FC_E_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == FC_E_UNSUPPORTED:
        raise UnsupportedError(f"{what}: {msg}")
    if rc == FC_E_CAPACITY:
        raise ValueError(f"{what}: capacity/workspace too small")
    raise CudaError(f"{what}: {msg}")


_cudart = None


def capture_probe(what: str) -> None:
    """Debug aid (FC_CAPTURE_CHECK=1): raise naming ``what`` if the current
    stream's graph capture has been invalidated by an earlier operation."""
    if not os.environ.get("FC_CAPTURE_CHECK"):
        return
    global _cudart
    import torch
    if _cudart is None:
        _cudart = ctypes.CDLL("libcudart.so.12")
    status = ctypes.c_int(0)
    _cudart.cudaStreamIsCapturing(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(status))
    if status.value == 2:  # cudaStreamCaptureStatusInvalidated
        raise RuntimeError(f"graph capture invalidated at or before: {what}")
