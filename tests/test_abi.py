"""CPU-side checks of the boundary: the C-ABI library loads and exports exactly
what include/sdfgi_b200.h declares; SDFS/SDFA round trips; struct layouts."""
import ctypes
import os
import re
import tempfile

import numpy as np

from golden_util import CASES, load
from paper_2007_14394_b200 import runtime, scene_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sdfgi_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"SDFGI_API\s+[\w\s\*]+?\b(sdfgi_\w+)\s*\(", src)))


def test_header_declares_the_binding_table():
    assert declared_symbols() == sorted(runtime.exported_symbols())


def test_library_loads_and_exports_every_declared_symbol():
    lib = runtime.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.sdfgi_abi_version() == 1


def test_no_device_means_loud_failure_not_fallback():
    n = runtime.device_count()
    if n == 0:
        try:
            runtime.Device(0)
        except runtime.SdfgiError as e:
            assert "no CUDA device" in str(e)
        else:
            raise AssertionError("context creation without a GPU must fail")


def test_struct_sizes_match_header():
    assert scene_io.PRIM_DTYPE.itemsize == 184
    assert scene_io.LIGHT_DTYPE.itemsize == 80
    assert scene_io.CLUSTER_DTYPE.itemsize == 56
    assert scene_io.CFG_DTYPE.itemsize == 224
    assert scene_io.PROBE_DTYPE.itemsize == 88
    assert scene_io.RAY_DTYPE.itemsize == 96


def test_sdfs_roundtrip_is_byte_exact():
    for name in CASES:
        path = os.path.join(ROOT, "tests", "golden", name, "scene.sdfs")
        s = scene_io.read_sdfs(path)
        with tempfile.TemporaryDirectory() as d:
            out = os.path.join(d, "x.sdfs")
            scene_io.write_sdfs(out, s)
            assert open(out, "rb").read() == open(path, "rb").read(), name


def test_sdfa_roundtrip():
    case = load("c1")
    a = case.data["atlas_p0_c0"]
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "a.sdfa")
        scene_io.write_sdfa(p, a)
        r, n, b = scene_io.read_sdfa(p)
        assert r == 8 and n == 512 and np.array_equal(a, b)
        assert os.path.getsize(p) == 16 + a.size * 4
