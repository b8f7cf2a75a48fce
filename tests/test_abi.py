"""CPU checks of the C-ABI library: it loads without a GPU and exports every function
include/ssnal_en.h declares; the binding mirrors the stats struct layout."""
import ctypes
import os
import re

import paper_2006_03970_b200 as pkg
from paper_2006_03970_b200 import ssnal_en as binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ssnal_en.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssnal_en_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(binding.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 12
    for nm in names:
        assert hasattr(lib, nm), nm


def test_version_and_error_without_gpu():
    lib = pkg.load_library()
    assert b"sm_100a" in lib.ssnal_en_version()
    assert isinstance(lib.ssnal_en_last_error(), bytes)


def test_stats_struct_layout_matches_header():
    # header: 10 int32 (incl. 3-array) + int64 + 8 doubles + int64 + double + 2 int32
    assert ctypes.sizeof(binding.Stats) == 10 * 4 + 8 + 8 * 8 + 8 + 8 + 2 * 4
    fields = [f for f, _ in binding.Stats._fields_]
    hdr = open(os.path.join(ROOT, "include", "ssnal_en.h")).read()
    body = hdr[hdr.index("typedef struct {"):hdr.index("} ssnal_en_stats;")]
    for f in fields:
        assert re.search(r"\b" + f + r"\b", body), f


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle or numpy-based compute paths."""
    for fn in os.listdir(os.path.join(ROOT, "paper_2006_03970_b200")):
        if fn.endswith(".py"):
            s = open(os.path.join(ROOT, "paper_2006_03970_b200", fn)).read()
            assert "oracle" not in s.replace("no CPU fallback", ""), fn
