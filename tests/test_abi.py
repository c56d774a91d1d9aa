"""CPU checks of the C-ABI boundary: libhive.so loads without a GPU and exports
every function include/hive.h declares; the product path has no route to the
oracle."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hive.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hive_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("hive_create", "hive_insert", "hive_find", "hive_erase", "hive_mixed", "hive_destroy"):
        assert n in names


def test_library_loads_and_exports_every_symbol():
    from paper_2510_15095_b200 import build, hive
    build.build()
    L = hive.lib()                            # loads on a GPU-less host (no libcuda link)
    out = subprocess.check_output(["nm", "-D", "--defined-only", hive.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (hive_[a-z0-9_]+)", out))
    for name in declared():
        assert name in exported, name
        assert name in hive.SIGNATURES, name   # the binding marshals every call
        getattr(L, name)
    # no torch / oracle symbols leak into the ABI
    assert not any("oracle" in s for s in exported)


def test_status_strings_without_gpu():
    from paper_2510_15095_b200 import hive
    L = hive.lib()
    assert L.hive_status_string(0) == b"ok"
    assert L.hive_status_string(5).startswith(b"stash full")
    # argument validation happens before any CUDA call
    assert L.hive_insert(None, None, None, 0, None, None) == 1      # NULL handle -> EINVAL
    assert L.hive_route(0, 0, None, None, None, 0, None, None, None, None, None) == 1
    assert L.hive_hash(7, None, 0, None, None) == 1                 # unknown hash fn
    y = hive._u64(0)
    assert L.hive_collisions(2, None, 0, 0, hive.ctypes.byref(y), None) == 1   # m = 0
    assert L.hive_gather_ceiling(None, 0, None, 1, None, None) == 1  # NULL blocks, n > 0
    assert L.hive_route_p2p(0, 0, 0, None, None, None, 0, 1, None, None, None, None, None, None) == 1
    assert L.hive_route_p2p(9, 0, 0, None, None, None, 0, 1, None, None, None, None, None, None) == 1
    assert L.hive_inbox_compact(9, 1, None, None, None, 0, None, None, None, None) == 1
    assert L.hive_return_p2p(2, 2, 1, None, 0, None, None, None, None, None) == 1   # rank >= n_src
    cfg = hive.HiveConfig()
    L.hive_config_default(hive.ctypes.byref(cfg))
    assert cfg.flags == 0                                           # default pair: BitHash1/2
    cfg.flags = 4                                                   # undefined flag bit
    h = hive.ctypes.c_void_p()
    assert L.hive_create(hive.ctypes.byref(cfg), None, hive.ctypes.byref(h)) == 1


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_15095_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "hive_oracle" not in txt, f
