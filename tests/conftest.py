"""Shared pytest setup.

Markers: `gpu` — needs a B200 (run with `-m gpu`); everything else runs on CPU.
The native libraries are (re)built in-tree on first use (tools/build.py).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import build  # tools/build.py

    build.build_synth()
    build.build_oracle()
    try:
        build.build_product()
    except Exception as e:  # product build problems surface in the ABI tests
        print("product build failed:", e)
    yield
