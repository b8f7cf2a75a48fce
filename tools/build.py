#!/usr/bin/env python3
"""Build every native artefact in-tree.

  synth/libsynth.so            host input generator      (gcc)
  synth/libsynth_cuda.so       device input generator    (nvcc, sm_100a)
  oracle/libssnal_oracle.so    CPU oracle (test infra)   (gcc, -ffp-contract=off)
  paper_2006_03970_b200/libssnal_en.so   the product C-ABI (nvcc, sm_100a)

Rebuilds only what is older than its sources unless force=True.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def build_synth(force=False):
    src = os.path.join(ROOT, "synth")
    host_srcs = [f"{src}/synth_host.c", f"{src}/gen_core.h"]
    out = f"{src}/libsynth.so"
    if force or _stale(out, host_srcs):
        _run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
              f"{src}/synth_host.c", "-o", out, "-lm"])
    dev_srcs = [f"{src}/synth_dev.cu", f"{src}/gen_core.h"]
    out = f"{src}/libsynth_cuda.so"
    if force or _stale(out, dev_srcs):
        _run([NVCC, *ARCH, "-O3", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "-shared", "-cudart", "static", f"{src}/synth_dev.cu", "-o", out])


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle")
    srcs = [f"{src}/ssnal_oracle.c"]
    out = f"{src}/libssnal_oracle.so"
    if os.path.exists(srcs[0]) and (force or _stale(out, srcs)):
        _run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
              srcs[0], "-o", out, "-lm"])


def build_product(force=False):
    pkg = os.path.join(ROOT, "paper_2006_03970_b200")
    csrc = os.path.join(pkg, "csrc")
    main = os.path.join(csrc, "ssnal_en.cu")
    if not os.path.exists(main):
        return
    srcs = glob.glob(f"{csrc}/*.cu") + glob.glob(f"{csrc}/*.cuh") + glob.glob(f"{ROOT}/include/*.h")
    out = os.path.join(pkg, "libssnal_en.so")
    if force or _stale(out, srcs):
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC",
              f"-I{ROOT}/include", "-shared", "-cudart", "static", main, "-o", out])


def build_all(force=False):
    if shutil.which(NVCC) is None and not os.path.exists(NVCC):
        raise RuntimeError("nvcc not found")
    build_synth(force)
    build_oracle(force)
    build_product(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
