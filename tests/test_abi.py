"""The C-ABI library: it builds for sm_100a, loads, exports every declared symbol,
and validates arguments without touching a GPU (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_0811_3448_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "binarsort_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    _lib.build()
    return _lib.lib()


def test_header_and_loader_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_library_is_sm100a(L):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tma_bulk_copies_in_sass(L):
    # the scatter/local kernels stream tiles with cp.async.bulk (SASS UBLKCP)
    sass = subprocess.run(["cuobjdump", "-sass", _lib.SO_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass


def test_version_and_workspace_sizes(L):
    assert L.bs_version() >= 100
    a = L.bs_workspace_bytes(1 << 20, 4, 0)
    b = L.bs_workspace_bytes(1 << 21, 4, 0)
    kv = L.bs_workspace_bytes(1 << 20, 4, 4)
    assert 0 < a < b and kv > a
    assert a >= 4 * (1 << 20)  # holds the ping-pong copy of the keys
    assert L.bs_workspace_bytes(16, 3, 0) == 0  # bad key width


def test_argument_errors_map_to_reference_exceptions(L):
    # validation happens before any CUDA call, so these run without a GPU
    rc = L.bs_sort(None, None, 10, 3, 0, 32, 0, 0, None, 0, None, None, 1)
    assert rc == _lib.BS_ERR_VALUE
    with pytest.raises(ValueError):
        _lib.check(rc)
    rc = L.bs_sort(None, None, 10, 4, 0, 33, 0, 0, None, 0, None, None, 1)  # width > word bits
    assert rc == _lib.BS_ERR_VALUE and b"width" in L.bs_last_error()
    rc = L.bs_sort(None, None, 10, 4, 0, 32, 33, 0, None, 0, None, None, 1)  # pos past width
    assert rc == _lib.BS_ERR_ASSERT
    with pytest.raises(AssertionError):
        _lib.check(rc)
    rc = L.bs_sort(None, None, 10, 4, 0, 32, 0, 2, None, 0, None, None, 1)  # float needs 64-bit words
    assert rc == _lib.BS_ERR_VALUE
    rc = L.bs_partition_words(None, None, 0, 4, 0, 32, 0, None, 0, None, None, None)  # empty range
    assert rc == _lib.BS_ERR_ASSERT
    rc = L.bs_partition_words(None, None, 5, 4, 0, 8, 8, None, 0, None, None, None)  # pos == width
    assert rc == _lib.BS_ERR_ASSERT
    rc = L.bs_split_by_splitters(None, None, 5, 4, 0, 32, 0, None, 9, None, None, None, None, 0, None)
    assert rc == _lib.BS_ERR_VALUE  # more than 8 ranks


def test_trivial_sorts_need_no_device(L):
    # n <= 1 and width 0 return before any launch (core.py:207-212)
    assert L.bs_sort(None, None, 1, 4, 0, 32, 0, 0, None, 0, None, None, 1) == _lib.BS_OK
    assert L.bs_sort(None, None, 0, 8, 8, 64, 0, 0, None, 0, None, None, 1) == _lib.BS_OK
    assert L.bs_sort(None, None, 100, 4, 0, 32, 32, 0, None, 0, None, None, 1) == _lib.BS_OK


def test_launch_accounting(L):
    assert L.bs_sort_launches(1, 4, 32, 0, 0) == 0
    small = L.bs_sort_launches(1000, 4, 32, 0, 0)
    big = L.bs_sort_launches(1 << 28, 4, 32, 0, 0)
    assert small == 3 and big > small
    assert L.bs_sort_launches(1 << 28, 4, 32, 0, 1) == big + 2
