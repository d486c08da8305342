"""``binarsort/_cuda.py``: the CUDA kernel module a reference maintainer adds.

A standalone ctypes binding of ``include/binarsort_b200.h`` (it does not
import ``paper_0811_3448_b200``) exposing the reference kernel-module ABI
(``/root/reference/pkg/src/binarsort/kernels.py:52-172``) with the same
names, arguments and counter semantics, so ``core``/``variants``/``bench``
run unchanged once ``kernels.py`` selects it.  Numpy
word arrays are copied to the device and back around each call; torch is
used only for device memory and the current stream.

Routing: ``sort_words`` with the baseline switches on a full-width range
from bit 0 takes the fast digit sort (``bs_sort``, counters by the closed
form); every other call -- the pass-through loop, the sortedness scan, a
start bit, words wider than ``width`` -- replays the reference's exact
permutations with ``bs_exact_sort`` (mode 0), and ``sort_words_iterative``
uses mode 1 (stack high-water mark).
"""

import ctypes
import os

import numpy as np

_LIB = os.environ.get("BINARSORT_CUDA_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_0811_3448_b200", "libbinarsort_b200.so")
_L = ctypes.CDLL(_LIB)
vp, u64, i32, i64, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
_LEVEL_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int)
_L.bs_last_error.restype = ctypes.c_char_p
_L.bs_workspace_bytes.argtypes = [u64, i32, i32]
_L.bs_workspace_bytes.restype = sz
_L.bs_sort.argtypes = [vp, vp, u64, i32, i32, i32, i32, i32, vp, sz, vp, vp, i64]
_L.bs_sort_status.argtypes = [vp, vp, vp]
_L.bs_partition_workspace_bytes.argtypes = [u64, i32, i32]
_L.bs_partition_workspace_bytes.restype = sz
_L.bs_partition_words.argtypes = [vp, vp, u64, i32, i32, i32, i32, vp, sz, vp, vp, vp]
_L.bs_range_sorted.argtypes = [vp, u64, i32, vp, vp]
_L.bs_exact_workspace_bytes.argtypes = [u64, i32, i32]
_L.bs_exact_workspace_bytes.restype = sz
_L.bs_exact_sort.argtypes = [vp, vp, u64, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i64,
                             vp, sz, vp, vp, _LEVEL_FN, vp]


def _check(rc):
    if rc == 0:
        return
    msg = _L.bs_last_error().decode(errors="replace")
    raise {1: ValueError, 2: AssertionError}.get(rc, RuntimeError)(msg)


def _torch():
    import torch

    return torch


def _dev(arr, lower, upper):
    t = _torch()
    view = np.ascontiguousarray(arr[lower:upper + 1])
    return t.from_numpy(view.view(np.int32 if arr.itemsize == 4 else np.int64)).cuda()


def _back(arr, lower, upper, d):
    arr[lower:upper + 1] = d.cpu().numpy().view(arr.dtype)


def _stream():
    return _torch().cuda.current_stream().cuda_stream


def _merge(counters, c):
    h = c.cpu().numpy()
    counters[0] += h[0]
    counters[1] += h[1]
    counters[2] += h[2]
    counters[3] = max(int(counters[3]), int(h[3]))


def new_counters():
    return np.zeros(4, dtype=np.int64)


def partition_words(arr, lower, upper, pos, width, counters):
    """kernels.partition_words (kernels.py:56-77): exact two-cursor permutation."""
    t = _torch()
    n = upper - lower + 1
    if n < 1:
        return lower
    d = _dev(arr, lower, upper)
    ws = t.empty(_L.bs_partition_workspace_bytes(n, arr.itemsize, 0), dtype=t.uint8, device="cuda")
    split = t.zeros(1, dtype=t.int64, device="cuda")
    c = t.zeros(4, dtype=t.int64, device="cuda")
    _check(_L.bs_partition_words(d.data_ptr(), None, n, arr.itemsize, 0, width, pos, ws.data_ptr(), ws.numel(),
                                 _stream(), split.data_ptr(), c.data_ptr()))
    _back(arr, lower, upper, d)
    _merge(counters, c)
    return lower + int(split.item())


def range_sorted_words(arr, lower, upper):
    """kernels.range_sorted_words (kernels.py:80-85)."""
    t = _torch()
    if upper <= lower:
        return True
    d = _dev(arr, lower, upper)
    flag = t.zeros(1, dtype=t.int32, device="cuda")
    _check(_L.bs_range_sorted(d.data_ptr(), upper - lower + 1, arr.itemsize, _stream(), flag.data_ptr()))
    return bool(int(flag.item()))


def _exact(arr, lower, upper, pos, width, mode, loop, check_after, streak, checked, depth, counters):
    t = _torch()
    n = upper - lower + 1
    d = _dev(arr, lower, upper)
    ws = t.empty(_L.bs_exact_workspace_bytes(n, arr.itemsize, 0), dtype=t.uint8, device="cuda")
    c = t.zeros(4, dtype=t.int64, device="cuda")
    _check(_L.bs_exact_sort(d.data_ptr(), None, n, arr.itemsize, 0, width, pos, 0, mode, int(bool(loop)),
                            int(check_after), int(streak), int(bool(checked)), 0, int(depth), ws.data_ptr(),
                            ws.numel(), _stream(), c.data_ptr(), _LEVEL_FN(), None))
    _back(arr, lower, upper, d)
    _merge(counters, c)


def sort_words(arr, lower, upper, pos, width, passthrough_loop, check_after, streak, checked, counters, depth):
    """kernels.sort_words (kernels.py:88-126)."""
    t = _torch()
    n = upper - lower + 1
    if n < 2 or pos >= width:  # the base case still counts one call (kernels.py:100-105)
        counters[2] += 1
        counters[3] = max(int(counters[3]), int(depth))
        return
    if passthrough_loop or check_after > 0 or pos > 0 or arr.itemsize * 8 != width:
        _exact(arr, lower, upper, pos, width, 0, passthrough_loop, check_after, streak, checked, depth, counters)
        return
    d = _dev(arr, lower, upper)
    ws = t.empty(_L.bs_workspace_bytes(n, arr.itemsize, 0), dtype=t.uint8, device="cuda")
    c = t.zeros(4, dtype=t.int64, device="cuda")
    st = t.zeros(1, dtype=t.int32, device="cuda")
    _check(_L.bs_sort(d.data_ptr(), None, n, arr.itemsize, 0, width, pos, 0, ws.data_ptr(), ws.numel(), _stream(),
                      c.data_ptr(), int(depth)))
    _check(_L.bs_sort_status(ws.data_ptr(), st.data_ptr(), _stream()))
    if int(st.item()):
        raise RuntimeError("device work-list overflow")
    _back(arr, lower, upper, d)
    _merge(counters, c)


def sort_words_iterative(arr, lower, upper, width, counters):
    """kernels.sort_words_iterative (kernels.py:129-172): max_depth = stack high-water mark."""
    n = upper - lower + 1
    if n < 1:  # the empty range is pushed once and passes through every bit
        counters[2] += width
        counters[3] = max(int(counters[3]), 1)
        return
    _exact(arr, lower, upper, 0, width, 1, False, 0, 0, False, 1, counters)
