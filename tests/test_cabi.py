"""CPU checks of the C-ABI boundary: libzpp.so loads and exports every symbol that
include/zpp.h declares (no compute calls - there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2402_03791_b200.engine import lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "zpp.h")


def declared() -> set[str]:
    txt = open(HEADER).read()
    return set(re.findall(r"\b(zpp_[a-z0-9_]+)\s*\(", txt))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(lib.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2402_03791_b200", "csrc"), "-j8"], check=True)
    return lib.load()


def test_header_declares_the_bound_api():
    assert declared() == set(lib.exported_symbols())


def test_library_exports_every_declared_symbol(so):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (zpp_[a-z0-9_]+)", out))
    assert declared() <= exported, declared() - exported


def test_pure_host_entry_points(so):
    assert so.zpp_version() == 1
    assert so.zpp_last_error() is not None
    # argument validation happens before any device work
    rc = so.zpp_gemm(None, 0, 7, None, 0, 8, None, 8, 0, 8, 8, 0, None, None, 0, None, 0, 0)
    assert rc == 1001 and b"empty" in so.zpp_last_error()
    rc = so.zpp_attn_fwd(None, None, None, 1, 100, 2, 64, 0)
    assert rc == 1001 and b"multiple of 128" in so.zpp_last_error()
    assert so.zpp_attn_bwd_workspace_floats(1, 128, 2, 64) == 2 * 2 * 128


def test_nccl_loads_from_torch_wheel(so):
    lib.load_nccl()
    buf = ctypes.create_string_buffer(128)
    assert so.zpp_nccl_unique_id(buf) == 0
