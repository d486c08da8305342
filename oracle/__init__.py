"""CPU oracle for the Binar Sort hot path -- TEST INFRASTRUCTURE ONLY.

This package is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  ``paper_0811_3448_b200`` never
imports it and has no CPU fallback.

``binarsort_oracle.c`` restates the reference numba kernels
(``/root/reference/pkg/src/binarsort/kernels.py``):

* ``partition_words``      -- kernels.py:56-77
* ``range_sorted_words``   -- kernels.py:80-85
* ``sort_words``           -- kernels.py:88-126
* ``sort_words_iterative`` -- kernels.py:129-172
* ``sort_parallel``        -- variants.py:162-229 (word path, pthreads pool)

Pinned against the reference's own known-answer tests and against vectors
produced by running the reference here (``tests/golden/make_golden.py``);
see ``tests/test_oracle_golden.py``.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "liboracle.so")

EXTRACTIONS, SWAPS, CALLS, MAX_DEPTH = 0, 1, 2, 3


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "binarsort_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, vp, ip = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        for suf in ("u32", "u64"):
            f = getattr(L, f"or_partition_words_{suf}")
            f.argtypes = [vp, i64, i64, i64, i64, vp]
            f.restype = i64
            f = getattr(L, f"or_range_sorted_words_{suf}")
            f.argtypes = [vp, i64, i64]
            f.restype = ip
            f = getattr(L, f"or_sort_words_{suf}")
            f.argtypes = [vp, i64, i64, i64, i64, ip, i64, i64, ip, vp, i64]
            f.restype = None
            f = getattr(L, f"or_sort_words_iterative_{suf}")
            f.argtypes = [vp, i64, i64, i64, vp]
            f.restype = None
        L.or_sort_parallel.argtypes = [vp, ip, i64, i64, i64, vp]
        L.or_sort_parallel.restype = ip
        _lib = L
    return _lib


def new_counters() -> np.ndarray:
    return np.zeros(4, dtype=np.int64)


def _suffix(arr: np.ndarray) -> str:
    if arr.dtype == np.uint32:
        return "u32"
    if arr.dtype == np.uint64:
        return "u64"
    raise TypeError(f"oracle handles uint32/uint64 words, got {arr.dtype}")


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data


def partition_words(arr, lower, upper, pos, width, counters) -> int:
    return int(getattr(lib(), f"or_partition_words_{_suffix(arr)}")(
        _ptr(arr), lower, upper, pos, width, _ptr(counters)))


def range_sorted_words(arr, lower, upper) -> bool:
    return bool(getattr(lib(), f"or_range_sorted_words_{_suffix(arr)}")(_ptr(arr), lower, upper))


def sort_words(arr, lower, upper, pos, width, passthrough_loop, check_after,
               streak, checked, counters, depth) -> None:
    getattr(lib(), f"or_sort_words_{_suffix(arr)}")(
        _ptr(arr), lower, upper, pos, width, int(bool(passthrough_loop)),
        check_after, streak, int(bool(checked)), _ptr(counters), depth)


def sort_words_iterative(arr, lower, upper, width, counters) -> None:
    getattr(lib(), f"or_sort_words_iterative_{_suffix(arr)}")(
        _ptr(arr), lower, upper, width, _ptr(counters))


def sort(arr: np.ndarray, width: int | None = None) -> np.ndarray:
    """core.sort word path (core.py:201-222): in place; returns counters."""
    if width is None:
        width = arr.dtype.itemsize * 8
    c = new_counters()
    if arr.size > 1 and width > 0:
        sort_words(arr, 0, arr.size - 1, 0, width, False, 0, 0, False, c, 1)
    return c


def sort_parallel(arr: np.ndarray, workers: int, width: int | None = None) -> np.ndarray:
    """variants.sort_parallel word path: in place; returns merged counters."""
    if width is None:
        width = arr.dtype.itemsize * 8
    m = new_counters()
    rc = lib().or_sort_parallel(_ptr(arr), int(arr.dtype == np.uint64), arr.size,
                                width, workers, _ptr(m))
    if rc != 0:
        raise ValueError("workers must be >= 1")
    return m
