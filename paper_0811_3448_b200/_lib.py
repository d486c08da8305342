"""Loader for the C-ABI library ``libbinarsort_b200.so`` (include/binarsort_b200.h).

The shared library is built in-tree by :func:`build` (``nvcc -gencode
arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if the library
is missing or no CUDA device is present, every sort entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
SO_PATH = os.path.join(_HERE, "libbinarsort_b200.so")
_CSRC = os.path.join(_HERE, "csrc")
_SOURCES = ["binarsort_b200.cu"]
_DEPS = sorted(f for f in os.listdir(_CSRC) if f.endswith((".cu", ".cuh"))) if os.path.isdir(_CSRC) else []

BS_OK, BS_ERR_VALUE, BS_ERR_ASSERT, BS_ERR_CUDA, BS_ERR_WORKSPACE, BS_ERR_INTERNAL = range(6)
BS_KEY_UNSIGNED, BS_KEY_SIGNED, BS_KEY_FLOAT = 0, 1, 2
EX_REC, EX_ITER, EX_LEVELS, EX_PAR = 0, 1, 2, 3  # bs_exact_sort modes
LEVEL_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int)  # bs_level_fn

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xcompiler", "-O3",
]

# every symbol include/binarsort_b200.h declares
EXPORTS = (
    "bs_version", "bs_last_error", "bs_workspace_bytes", "bs_sort",
    "bs_metrics_workspace_bytes", "bs_metrics", "bs_partition_workspace_bytes",
    "bs_partition_words", "bs_range_sorted", "bs_split_workspace_bytes",
    "bs_split_by_splitters", "bs_sample_keys", "bs_sort_profiled", "bs_sort_launches",
    "bs_sort_from_workspace_bytes", "bs_sort_from", "bs_split_count", "bs_split_exchange",
    "bs_ipc_handle_bytes", "bs_ipc_alloc", "bs_ipc_open", "bs_ipc_close", "bs_ipc_free",
    "bs_sort_status", "bs_debug_capacity", "bs_exact_workspace_bytes", "bs_exact_sort",
    "bs_exact_boundaries", "bs_debug_checks", "bs_exact_snapshot", "bs_sort_status_offset",
)


SO_DEBUG_PATH = os.path.join(_HERE, "libbinarsort_b200_debug.so")  # -DBS_DEBUG_CHECKS build


def _stale(path: str) -> bool:
    if not os.path.exists(path):
        return True
    so_m = os.path.getmtime(path)
    deps = [os.path.join(_CSRC, d) for d in _DEPS]
    deps.append(os.path.join(_ROOT, "include", "binarsort_b200.h"))
    return any(os.path.exists(d) and os.path.getmtime(d) > so_m for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = True) -> str:
    """Compile the CUDA library in-tree for sm_100a (no GPU needed).

    Also builds the bounds-checked variant (``-DBS_DEBUG_CHECKS``) that the
    test suite runs its parity corpus against (``BS_LIBRARY=debug``).
    """
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.isabs(nvcc) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    jobs = [(SO_PATH, [])] + ([(SO_DEBUG_PATH, ["-DBS_DEBUG_CHECKS"])] if debug else [])
    procs = []
    for path, extra in jobs:
        if force or _stale(path):
            cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", path + ".tmp", *[os.path.join(_CSRC, s) for s in _SOURCES]]
            if verbose:
                print(" ".join(cmd))
            procs.append((path, subprocess.Popen(cmd)))
    for path, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc")
        os.replace(path + ".tmp", path)
    return SO_PATH


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """The loaded library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        which = os.environ.get("BS_LIBRARY", "")
        # "debug": the bounds-checked build; a path: a scratch build (kernel experiments)
        path = SO_DEBUG_PATH if which == "debug" else (which if which.endswith(".so") else SO_PATH)
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = ctypes.CDLL(path)
        vp, u64, i32, i64, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        L.bs_version.restype = i32
        L.bs_debug_checks.restype = i32
        L.bs_last_error.restype = ctypes.c_char_p
        L.bs_workspace_bytes.argtypes = [u64, i32, i32]
        L.bs_workspace_bytes.restype = sz
        L.bs_sort.argtypes = [vp, vp, u64, i32, i32, i32, i32, i32, vp, sz, vp, vp, i64]
        L.bs_sort.restype = i32
        L.bs_metrics_workspace_bytes.argtypes = [u64]
        L.bs_metrics_workspace_bytes.restype = sz
        L.bs_metrics.argtypes = [vp, u64, i32, i32, i32, i32, i64, vp, sz, vp, vp]
        L.bs_metrics.restype = i32
        L.bs_partition_workspace_bytes.argtypes = [u64, i32, i32]
        L.bs_partition_workspace_bytes.restype = sz
        L.bs_partition_words.argtypes = [vp, vp, u64, i32, i32, i32, i32, vp, sz, vp, vp, vp]
        L.bs_partition_words.restype = i32
        L.bs_range_sorted.argtypes = [vp, u64, i32, vp, vp]
        L.bs_range_sorted.restype = i32
        L.bs_split_workspace_bytes.argtypes = [u64, i32, i32, i32]
        L.bs_split_workspace_bytes.restype = sz
        L.bs_split_by_splitters.argtypes = [vp, vp, u64, i32, i32, i32, i32, vp, i32, vp, vp, vp, vp, sz, vp]
        L.bs_split_by_splitters.restype = i32
        L.bs_sample_keys.argtypes = [vp, u64, i32, i32, i32, u64, vp, vp]
        L.bs_sample_keys.restype = i32
        L.bs_sort_profiled.argtypes = [vp, vp, u64, i32, i32, i32, i32, i32, vp, sz, vp, vp, i64,
                                       ctypes.POINTER(ctypes.c_float), i32, ctypes.POINTER(i32)]
        L.bs_sort_profiled.restype = i32
        L.bs_sort_launches.argtypes = [u64, i32, i32, i32, i32]
        L.bs_sort_launches.restype = i32
        L.bs_sort_from_workspace_bytes.argtypes = [u64, i32, i32]
        L.bs_sort_from_workspace_bytes.restype = sz
        L.bs_sort_from.argtypes = [vp, vp, vp, vp, u64, i32, i32, i32, i32, i32, vp, sz, vp]
        L.bs_sort_from.restype = i32
        L.bs_split_count.argtypes = [vp, u64, i32, i32, i32, vp, i32, vp, vp, sz, vp]
        L.bs_split_count.restype = i32
        L.bs_split_exchange.argtypes = [vp, vp, u64, i32, i32, i32, i32, vp, i32, vp, vp, vp, vp, vp, sz, vp]
        L.bs_split_exchange.restype = i32
        L.bs_ipc_handle_bytes.restype = sz
        L.bs_ipc_alloc.argtypes = [sz, ctypes.POINTER(vp), vp]
        L.bs_ipc_alloc.restype = i32
        L.bs_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
        L.bs_ipc_open.restype = i32
        L.bs_ipc_close.argtypes = [vp]
        L.bs_ipc_close.restype = i32
        L.bs_ipc_free.argtypes = [vp]
        L.bs_ipc_free.restype = i32
        L.bs_sort_status.argtypes = [vp, vp, vp]
        L.bs_sort_status.restype = i32
        L.bs_sort_status_offset.restype = sz
        L.bs_debug_capacity.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.bs_debug_capacity.restype = None
        L.bs_exact_workspace_bytes.argtypes = [u64, i32, i32]
        L.bs_exact_workspace_bytes.restype = sz
        L.bs_exact_sort.argtypes = [vp, vp, u64, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i64,
                                    vp, sz, vp, vp, LEVEL_FN, vp]
        L.bs_exact_sort.restype = i32
        L.bs_exact_boundaries.argtypes = [vp, u64, i32, i32, vp, vp, vp]
        L.bs_exact_boundaries.restype = i32
        L.bs_exact_snapshot.argtypes = [vp, vp, u64, i32, i32, i32, vp, vp]
        L.bs_exact_snapshot.restype = i32
        _lib = L
        return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == BS_OK:
        return
    msg = lib().bs_last_error().decode(errors="replace")
    if rc == BS_ERR_VALUE:
        raise ValueError(msg)
    if rc == BS_ERR_ASSERT:
        raise AssertionError(msg)
    raise RuntimeError(f"binarsort_b200 error {rc}: {msg}")
