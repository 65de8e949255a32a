"""Shared pytest setup: repo on sys.path, `gpu` marker, in-tree build of the native libraries.

`-m "not gpu"` tests run here on CPU (oracle pins, generator, host logic, C-ABI symbol exports);
`-m gpu` tests are the CUDA-vs-oracle parity tests and need a B200.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


_built = set()


def build(target: str):
    """Incremental in-tree `make <target>` (no-op when up to date)."""
    if target in _built:
        return
    subprocess.run(["make", "-s", "-C", ROOT, target], check=True)
    _built.add(target)


@pytest.fixture(scope="session", autouse=True)
def _native_libs():
    build("gen")
    build("oracle")
    yield
