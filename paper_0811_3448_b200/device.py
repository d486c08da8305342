"""Device plumbing: torch CUDA buffers, streams and workspaces around the C ABI.

PyTorch is used only for device memory, the current stream and (in
``dist.py``) ``torch.distributed``; every byte of sorting work runs in
``libbinarsort_b200.so``.  There is no CPU fallback: without a CUDA device the
entry points raise ``RuntimeError``.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_NP_WORD = {4: np.uint32, 8: np.uint64}


def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("binarsort_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return t


def is_torch_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


_RAW = None


def _raw_dtype(itemsize: int):
    """torch dtype used as raw word storage of the given byte width."""
    t = torch()
    return {4: t.int32, 8: t.int64}[itemsize]


def as_raw_words(x):
    """View a 1-D torch tensor of 4/8-byte elements as int32/int64 raw words."""
    t = torch()
    if x.element_size() not in (4, 8):
        raise TypeError(f"word arrays need 4- or 8-byte elements, got {x.dtype}")
    want = _raw_dtype(x.element_size())
    return x if x.dtype == want else x.view(want)


def stream_ptr(device=None) -> int:
    t = torch()
    return t.cuda.current_stream(device).cuda_stream


class _WorkspaceCache:
    """Per-device grow-only workspace (a torch uint8 tensor from the caching allocator)."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, device):
        t = torch()
        dev = t.device(device)
        key = dev.index if dev.index is not None else t.cuda.current_device()
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=dev)
            self._bufs[key] = buf
        return buf

    def clear(self):
        self._bufs.clear()


workspaces = _WorkspaceCache()


def sort_words_device(keys, vals=None, *, width: int, start_pos: int = 0, key_kind: int = 0,
                      counters=None, depth: int = 1, workspace=None):
    """Sort a contiguous 1-D CUDA tensor of raw words in place (bs_sort).

    ``counters``: optional CUDA int64[4] tensor receiving the reference Metrics.
    ``workspace``: optional CUDA uint8 tensor (defaults to the per-device cache).
    """
    t = require_cuda()
    if not keys.is_cuda or keys.dim() != 1 or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous 1-D CUDA tensor")
    n = keys.numel()
    kb = keys.element_size()
    vb = 0
    vptr = None
    if vals is not None:
        if not vals.is_cuda or vals.dim() != 1 or not vals.is_contiguous() or vals.numel() != n:
            raise ValueError("values must be a contiguous 1-D CUDA tensor of the same length")
        vb = vals.element_size()
        vptr = vals.data_ptr()
    L = _lib.lib()
    need = L.bs_workspace_bytes(n, kb, vb)
    if workspace is None:
        workspace = workspaces.get(need, keys.device)
    elif workspace.numel() < need:
        raise ValueError(f"workspace too small: need {need} bytes")
    cptr = None
    if counters is not None:
        if counters.dtype != t.int64 or counters.numel() != 4 or not counters.is_cuda:
            raise ValueError("counters must be a CUDA int64[4] tensor")
        cptr = counters.data_ptr()
    with t.cuda.device(keys.device):
        rc = L.bs_sort(keys.data_ptr(), vptr, n, kb, vb, int(width), int(start_pos), int(key_kind),
                       workspace.data_ptr(), workspace.numel(), stream_ptr(keys.device), cptr, int(depth))
    _lib.check(rc)


def metrics_device(sorted_keys, *, width: int, start_pos: int = 0, key_kind: int = 0, depth: int = 1,
                   counters):
    """Add the closed-form reference Metrics of an already sorted CUDA word tensor."""
    t = require_cuda()
    L = _lib.lib()
    with t.cuda.device(sorted_keys.device):
        rc = L.bs_metrics(sorted_keys.data_ptr(), sorted_keys.numel(), sorted_keys.element_size(), int(width),
                          int(start_pos), int(key_kind), int(depth), None, 0, stream_ptr(sorted_keys.device),
                          counters.data_ptr())
    _lib.check(rc)


def partition_device(keys, vals=None, *, width: int, pos: int, counters=None):
    """Exact reference partition pass on a contiguous CUDA word tensor; returns split (device)."""
    t = require_cuda()
    L = _lib.lib()
    n = keys.numel()
    kb = keys.element_size()
    vb = vals.element_size() if vals is not None else 0
    ws = workspaces.get(L.bs_partition_workspace_bytes(n, kb, vb), keys.device)
    split = t.zeros(1, dtype=t.int64, device=keys.device)
    with t.cuda.device(keys.device):
        rc = L.bs_partition_words(keys.data_ptr(), vals.data_ptr() if vals is not None else None, n, kb, vb,
                                  int(width), int(pos), ws.data_ptr(), ws.numel(), stream_ptr(keys.device),
                                  split.data_ptr(), counters.data_ptr() if counters is not None else None)
    _lib.check(rc)
    return split


def range_sorted_device(keys) -> bool:
    t = require_cuda()
    L = _lib.lib()
    flag = t.zeros(1, dtype=t.int32, device=keys.device)
    with t.cuda.device(keys.device):
        rc = L.bs_range_sorted(keys.data_ptr(), keys.numel(), keys.element_size(), stream_ptr(keys.device),
                               flag.data_ptr())
    _lib.check(rc)
    return bool(int(flag.item()))


def to_device_words(arr: np.ndarray, device="cuda"):
    """Upload a host word array (any 1-D view) as a contiguous raw-word CUDA tensor."""
    t = require_cuda()
    a = np.ascontiguousarray(arr)
    raw = a.view({4: np.int32, 8: np.int64}[a.dtype.itemsize])
    return t.from_numpy(raw).to(device, non_blocking=False)


def to_host_words(dev, out: np.ndarray) -> None:
    """Copy a raw-word CUDA tensor back into a host array view (handles strides)."""
    host = dev.cpu().numpy()
    out[...] = host.view(out.dtype)
