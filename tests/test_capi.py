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
    # 10 int32 geometry fields then 10 pointers
    assert ctypes.sizeof(_lib.FcStore) == 10 * 4 + 10 * 8
    assert _lib.FcStore.kv_pool.offset == 40


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
