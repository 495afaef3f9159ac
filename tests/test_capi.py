"""CPU checks of the C-ABI boundary: the in-tree library loads (no GPU
needed to dlopen it) and exports every symbol the header declares; the
ctypes struct mirrors the C struct layout."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2511_00868_b200 import _lib


def test_library_present_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run `make` / __graft_entry__.build() first"
    lib = _lib.load()
    assert lib.fc_version().decode().startswith("flexicache-b200")


def test_every_header_symbol_is_exported():
    declared = _lib.header_symbols()
    assert len(declared) >= 15
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(fc_\w+)", nm))
    assert set(declared) <= exported
    assert set(declared) == set(_lib._SIGNATURES)  # every entry point has a prototype


def test_struct_layout_matches_header():
    # 10 int32 geometry fields then 10 buffer pointers, then the optional
    # per-request state (row_phase, row_hold, stats)
    assert ctypes.sizeof(_lib.FcStore) == 10 * 4 + 13 * 8
    assert _lib.FcStore.kv_pool.offset == 40
    assert _lib.FcStore.row_phase.offset == 40 + 10 * 8
    assert _lib.FcStore.stats.offset == 40 + 12 * 8


def test_argument_errors_map_to_valueerror_without_gpu():
    """Synchronous validation happens before any CUDA call."""
    lib = _lib.load()
    rc = lib.fc_select_topk(None, 4, None, 1, 0, 1, None, None, None)  # k < 1
    with pytest.raises(ValueError, match="k must be >= 1"):
        _lib.check(rc, "fc_select_topk")
    rc = lib.fc_alloc_pages(None, 0, 0, 1, None)
    with pytest.raises(ValueError, match="null store"):
        _lib.check(rc, "fc_alloc_pages")


def test_unsupported_geometry_rejected():
    lib = _lib.load()
    s = _lib.FcStore(1, 1, 1, 1, 96, 16, 4, 4, 0, 8, *([1] * 10))  # d = 96 not compiled
    rc = lib.fc_step_advance(ctypes.byref(s), 1, None)
    with pytest.raises(ValueError, match="head_dim 96"):
        _lib.check(rc, "fc_step_advance")


def _fake_store(**kw):
    """A valid-looking descriptor (non-null dummy pointers): argument checks
    run, no kernel is launched."""
    geo = dict(batch_cap=2, layers=4, kv_heads=2, group=4, head_dim=128, page_size=16, pages_cap=64,
               sel_cap=16, dtype=_lib.FC_BF16, n_blocks=128)
    geo.update(kw)
    return _lib.FcStore(*geo.values(), *([64] * 10))


@pytest.mark.parametrize("call,msg", [
    (lambda lib, s: lib.fc_sparse_decode_layers(s, 3, 2, 64, 0, None, None, 0, 64, 0, None, 0, 0.1, 1, 0, 0,
                                                8, 64, 1 << 20, 1, None), "layer run out of range"),
    (lambda lib, s: lib.fc_sparse_decode_layers(s, 0, 2, 64, 0, None, None, 0, 64, 0, None, 0, 0.1, 1, 0, 0,
                                                8, 64, 1 << 20, 1, None), "layer strides"),
    (lambda lib, s: lib.fc_sparse_decode_layers(s, 0, 1, 64, 0, None, None, 0, 64, 0, None, 0, -1.0, 1, 0, 0,
                                                8, 64, 1 << 20, 1, None), "scale must be positive"),
    (lambda lib, s: lib.fc_score_attend(s, 9, 64, 64, 4, 0, 8, 1, 0, 64, None, None, 64, None, 0.1, 0, 1, None),
     "layer out of range"),
    (lambda lib, s: lib.fc_score_attend(s, 0, 64, 64, 0, 0, 8, 1, 0, 64, None, None, 64, None, 0.1, 0, 1, None),
     "period must be >= 1"),
    (lambda lib, s: lib.fc_score_attend(s, 0, 64, 64, 4, 0, 8, 1, 0, 64, 64, None, 64, None, 0.1, 0, 1, None),
     "k_new and v_new go together"),
    (lambda lib, s: lib.fc_free_row(s, 5, None), "row out of range"),
    (lambda lib, s: lib.fc_stage_plan(s, 64, 64, 64, 64, 64, 64, 64, 0, 1, 0, None), "capacity must be >= 1"),
    (lambda lib, s: lib.fc_stage_fetch(s, 64, 64, 64, 8, 64, 7, None), "pass must be in 0..3"),
    (lambda lib, s: lib.fc_fetch_pages_staged(s, 0, 64, 64, 64, 8, None, 64, None, None), "null buffer"),
    (lambda lib, s: lib.fc_offload_pages_ctas(s, 64, 64, 4, -1, None), "max_ctas must be >= 0"),
    (lambda lib, s: lib.fc_rerank_recycle_rows(s, 9, 64, 64, 64, 4, 0, 0, 1, None, 64, 64, 8, 64, 64, 1, None),
     "layer out of range"),
    (lambda lib, s: lib.fc_rerank_recycle_rows(s, 0, 64, 64, 64, 0, 0, 0, 1, None, 64, 64, 8, 64, 64, 1, None),
     "period must be >= 1"),
])
def test_new_entry_points_validate_without_gpu(call, msg):
    lib = _lib.load()
    s = _fake_store()
    rc = call(lib, ctypes.byref(s))
    with pytest.raises(ValueError, match=msg):
        _lib.check(rc, "call")
