"""The drop-in boundary: libtomograd_b200.so loads, exports every entry point
include/tomograd_b200.h declares, and fails loudly (no CPU fallback) when no
CUDA device is visible."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tomograd_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ["tg_cone_backproject", "tg_cone_forward", "tg_cone_fdk", "tg_planar_forward",
              "tg_planar_backproject", "tg_filter_apply", "tg_make_cone", "tg_last_error"]:
        assert s in syms
    assert len(syms) >= 40


def test_library_exports_every_declared_symbol(tg):
    lib = C.CDLL(tg._native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header(tg):
    assert set(declared_symbols()) == set(tg._native.SIGNATURES)


def test_abi_version(tg):
    assert tg._native.lib().tg_abi_version() == 1


def test_no_cpu_fallback_without_device(tg):
    import math
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is visible")
    vol = tg.VolumeSpec.centered([8, 8, 8], [1.0] * 3)
    geo = tg.make_cone(vol, tg.Detector2D.centered(8, 8, 1, 1), 4, math.pi, 50.0, 100.0)
    with pytest.raises(tg.CudaError, match="no CUDA device"):
        geo._plan(0)
    # host-buffer operators go through the same plan: they must raise too
    import numpy as np
    with pytest.raises(tg.CudaError):
        tg.forward_project(tg.Image(vol, np.zeros((8, 8, 8), np.float32)), geo)


def test_exports_are_c_abi():
    """extern "C" names (no C++ mangling) for every tg_* symbol"""
    out = os.popen(f"nm -D --defined-only {os.path.join(ROOT, 'paper_1904_13342_b200', 'libtomograd_b200.so')}").read()
    names = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for s in declared_symbols():
        assert s in names
