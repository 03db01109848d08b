"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library builds and loads,
exports every function include/evoke.h declares, validates arguments before touching the
device, and the product package never reaches the oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evoke.h")


@pytest.fixture(scope="module")
def pkg():
    from paper_1911_10616_b200 import build
    build.build()
    import paper_1911_10616_b200 as p
    p.lib()
    return p


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(evoke_[a-z_]+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = _declared_functions()
    assert {"evoke_orbits_edges", "evoke_orbits_csr", "evoke_orbits_edges_multi", "evoke_default_options",
            "evoke_strerror",
            "evoke_last_error", "evoke_version", "evoke_pass_name"} <= set(names)
    assert "#define EVOKE_NUM_ORBITS 73" in open(HEADER).read()


def test_library_exports_every_declared_symbol(pkg):
    out = subprocess.check_output(["nm", "-D", "--defined-only", pkg.LIB_PATH]).decode()
    exported = set(re.findall(r"\sT\s+(\w+)", out))
    missing = [f for f in _declared_functions() if f not in exported]
    assert not missing, missing
    assert set(pkg.EXPORTED_SYMBOLS) <= exported


def test_library_is_sm100a(pkg):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_version_strerror_passes(pkg):
    assert "sm100a" in pkg.version()
    L = pkg.lib()
    assert L.evoke_strerror(0) == b"ok"
    assert L.evoke_strerror(-1) == b"invalid argument"
    names = pkg.pass_names()
    assert len(names) == 16 and names[0] == "h2d" and names[-1] == "d2h"


def test_argument_validation_without_gpu(pkg):
    L = pkg.lib()
    o = pkg._Options()
    L.evoke_default_options(ctypes.byref(o))
    assert o.induced == 1 and o.num_shards == 1 and o.device == -1
    out = np.zeros((4, 73), np.uint64)
    e = np.zeros((1, 2), np.int32)
    assert L.evoke_orbits_edges(-1, 0, None, out.ctypes.data, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert L.evoke_orbits_edges(4, -2, e.ctypes.data, out.ctypes.data, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert L.evoke_orbits_edges(4, 3, None, out.ctypes.data, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert L.evoke_orbits_edges(4, 1, e.ctypes.data, None, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert L.evoke_orbits_edges(1 << 31, 1, e.ctypes.data, out.ctypes.data, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert b"bad n" in L.evoke_last_error()
    o2 = pkg._Options()
    L.evoke_default_options(ctypes.byref(o2))
    o2.num_shards = 2
    o2.shard_index = 2
    assert L.evoke_orbits_edges(4, 1, e.ctypes.data, out.ctypes.data, ctypes.byref(o2)) == pkg.EVOKE_EINVAL
    # n = 0 is a valid empty problem
    assert L.evoke_orbits_edges(0, 0, None, None, ctypes.byref(o)) == pkg.EVOKE_OK
    # malformed CSR (host pointers are validated on the host)
    rp = np.array([0, 2, 1, 3], np.int64)
    col = np.zeros(3, np.int32)
    out3 = np.zeros((3, 73), np.uint64)
    assert L.evoke_orbits_csr(3, rp.ctypes.data, col.ctypes.data, out3.ctypes.data,
                              ctypes.byref(o)) == pkg.EVOKE_EINVAL
    rp = np.array([1, 2, 2, 3], np.int64)
    assert L.evoke_orbits_csr(3, rp.ctypes.data, col.ctypes.data, out3.ctypes.data,
                              ctypes.byref(o)) == pkg.EVOKE_EINVAL
    with pytest.raises(pkg.EvokeError):
        pkg.evoke_orbits_edges(4, e, num_shards=0)
    # several GPUs in one process: the device list and the shard arguments are checked first
    devs = (ctypes.c_int * 2)(0, 0)
    M = L.evoke_orbits_edges_multi
    assert M(4, 1, e.ctypes.data, out.ctypes.data, None, 2, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(4, 1, e.ctypes.data, out.ctypes.data, devs, 0, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(4, 1, e.ctypes.data, out.ctypes.data, devs, 65, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(4, 1, e.ctypes.data, out.ctypes.data, devs, 2, ctypes.byref(o2)) == pkg.EVOKE_EINVAL
    assert M(-1, 1, e.ctypes.data, out.ctypes.data, devs, 2, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(4, 1, None, out.ctypes.data, devs, 2, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(4, 1, e.ctypes.data, None, devs, 2, ctypes.byref(o)) == pkg.EVOKE_EINVAL
    assert M(0, 0, None, None, devs, 2, ctypes.byref(o)) == pkg.EVOKE_OK
    # the kept scratch: bad ordinal rejected; releasing when nothing is kept is a no-op
    assert L.evoke_release_scratch(64) == pkg.EVOKE_EINVAL
    assert L.evoke_release_scratch(-2) == pkg.EVOKE_EINVAL
    assert L.evoke_release_scratch(-1) == pkg.EVOKE_OK


def test_binding_fails_loudly_without_library(pkg, monkeypatch):
    monkeypatch.setattr(pkg, "_lib", None)
    monkeypatch.setattr(pkg, "LIB_PATH", "/nonexistent/libevoke.so")
    with pytest.raises(ImportError):
        pkg.evoke_orbits_edges(3, np.array([[0, 1]], np.int32))


def test_product_never_reaches_the_oracle():
    pkgdir = os.path.join(ROOT, "paper_1911_10616_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, flags=re.M), f
                assert "evoke_oracle" not in text and "liboracle" not in text, f


def test_oracle_shares_no_source_with_product():
    orc = open(os.path.join(ROOT, "oracle", "evoke_oracle.c")).read()
    assert "#include" in orc
    for inc in re.findall(r'#include\s+"([^"]+)"', orc):
        assert "paper_1911_10616_b200" not in inc and "csrc" not in inc
