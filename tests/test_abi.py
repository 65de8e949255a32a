"""C-ABI checks that need no GPU: libsx.so builds for sm_100a, loads, and exports every
function include/sx.h declares; the binding mirrors the header's struct sizes."""
import ctypes
import os
import re
import subprocess

import pytest

from tests.conftest import ROOT, build


@pytest.fixture(scope="module")
def libsx():
    build("sx")
    from paper_2508_04701_b200 import _abi

    return _abi, ctypes.CDLL(_abi.LIB_PATH)


def header_functions():
    src = open(os.path.join(ROOT, "include", "sx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sx_status|void|int64_t|uint32_t|int|const char\*)\s+(sx_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("sx_filter", "sx_hash_build", "sx_hash_probe", "sx_groupby_agg", "sx_sort_topk"):
        assert f in fns


def test_every_declared_symbol_is_exported(libsx):
    _abi, L = libsx
    fns = header_functions()
    assert sorted(_abi.EXPORTS) == fns
    for f in fns:
        assert hasattr(L, f), f


def test_sm100a_code_in_library(libsx):
    _abi, _ = libsx
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_header(libsx):
    _abi, _ = libsx
    # sizes fixed by include/sx.h layout (x86-64): keep the binding in lock-step
    assert ctypes.sizeof(_abi.Col) == 40
    assert ctypes.sizeof(_abi.Sel) == 16
    assert ctypes.sizeof(_abi.Factor) == 24
    assert ctypes.sizeof(_abi.Term) == 88
    assert ctypes.sizeof(_abi.Expr) == 184
    assert ctypes.sizeof(_abi.Pred) == 40
    assert ctypes.sizeof(_abi.Agg) == 192
    assert ctypes.sizeof(_abi.TpchTables) == 40 * 24
    assert ctypes.sizeof(_abi.Q1Row) == 8 + 4 * 16 + 3 * 8 + 8


def test_no_device_means_loud_failure(libsx):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2508_04701_b200 as sx

    with pytest.raises(sx.SxError):
        sx.Ctx()
