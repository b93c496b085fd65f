"""CPU-side checks of the C-ABI library: it builds, loads, and exports every symbol that
include/dc.h declares. No compute calls (no GPU here)."""
import ctypes
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    from paper_2411_02797_b200 import build, _lib
    build.build()
    L = ctypes.CDLL(_lib.SO_PATH)
    names = _lib.exported_symbols()
    assert "dc_cct_build" in names and "dc_cct_merge_ranks" in names and len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the binding declares a signature for each of them
    _lib.lib()


def test_struct_layouts_match_header():
    from paper_2411_02797_b200 import _lib
    assert ctypes.sizeof(_lib.dc_topk_entry) == 24
    assert ctypes.sizeof(_lib.dc_paths) == 24
    assert ctypes.sizeof(_lib.dc_diag) == 64


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2411_02797_b200 as dc
    with pytest.raises(RuntimeError):
        dc.Context(0)


def test_sass_is_sm100a():
    from paper_2411_02797_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
