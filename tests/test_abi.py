"""CPU checks of the C-ABI library: it loads without a GPU and exports every function
include/ssnal_en.h declares; the binding mirrors the stats struct layout."""
import ctypes
import os
import re

import pytest

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


def _c_layout(struct, fields):
    """sizeof and offsetof of a header struct, compiled with gcc from include/ssnal_en.h."""
    import subprocess
    import tempfile
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"ssnal_en.h\"\nint main(void){printf(\"%zu\", sizeof(" + struct + "));"
    for f in fields:
        src += 'printf(" %zu", offsetof(' + struct + ", " + f + "));"
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    return int(out[0]), [int(v) for v in out[1:]]


@pytest.mark.parametrize("name,cls", [("ssnal_en_stats", "Stats"), ("ssnal_en_criteria", "Criteria")])
def test_struct_layout_matches_header(name, cls):
    """ctypes mirrors have the header's size and every field at the header's offset."""
    C = getattr(binding, cls)
    fields = [f for f, _ in C._fields_]
    size, offs = _c_layout(name, fields)
    assert ctypes.sizeof(C) == size
    for f, off in zip(fields, offs):
        assert getattr(C, f).offset == off, f



def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle or numpy-based compute paths."""
    for fn in os.listdir(os.path.join(ROOT, "paper_2006_03970_b200")):
        if fn.endswith(".py"):
            s = open(os.path.join(ROOT, "paper_2006_03970_b200", fn)).read()
            assert "oracle" not in s.replace("no CPU fallback", ""), fn
