"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/inpc_raster.h declares, and reports argument errors synchronously
(no compute calls are made here)."""
import ctypes as ct
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def m():
    from paper_2508_19140_b200 import build
    build.build()
    import paper_2508_19140_b200 as m
    return m


def declared_symbols():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"INPC_API\s+[\w\s\*]+?\b(inpc_\w+)\s*\(", txt))
    return names


def test_exports_every_declared_symbol(m):
    names = declared_symbols()
    assert len(names) >= 10
    lib = ct.CDLL(m.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(m.EXPORTS) == names


def test_library_is_sm100a(m):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", m.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_null_ctx(m):
    assert "inpc_raster" in m.version()
    assert m.lib.inpc_status_string(m.INVALID_ARG).decode() == "invalid argument"
    cfg = m.make_cfg(64, 64, 4)
    rc = m.lib.inpc_rasterize_fwd(None, ct.byref(cfg), None, 1, None, None, 0, None, 0, None, 0,
                                  None, None, None, None, None, None)
    assert rc == m.INVALID_ARG
    rc = m.lib.inpc_rasterize_bwd(None, ct.byref(cfg), None, 1, None, None, 0, None, 0, None, 0,
                                  None, None, None, None, None, None)
    assert rc == m.INVALID_ARG
    assert m.lib.inpc_stage_name(0).decode() == "memset"
    assert m.lib.inpc_stage_name(99) is None


def test_struct_layouts_match_header(m):
    # inpc_camera: 9+3+5 floats; inpc_raster_cfg: 4 ints, 4 floats, 2 ints, 1 uint, 2 ints
    assert ct.sizeof(m.Camera) == 17 * 4
    assert ct.sizeof(m.RasterCfg) == 13 * 4


def test_no_oracle_in_product_path():
    """The product package never imports / links the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2508_19140_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "inpc_oracle" not in txt and "liboracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2508_19140_b200", txt, re.M), f
            assert not re.search(r'#include\s+"[^"]*(inpc_raster|kernels|raster_math)', txt), f
