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
    """Grow-only workspaces keyed by (device, stream), guarded by a lock.

    A sort's workspace is live until its kernels finish, so two sorts in
    flight on different streams (pool threads, like the reference's
    ``sort_parallel`` workers, variants.py:195-206) must not share one: each
    (device, stream) pair gets its own buffer, allocated on that stream so the
    caching allocator orders its reuse with the stream's work.
    """

    def __init__(self):
        import threading

        self._bufs = {}
        self._lock = threading.Lock()

    def get(self, nbytes: int, device, stream=None):
        t = torch()
        dev = t.device(device)
        idx = dev.index if dev.index is not None else t.cuda.current_device()
        if stream is None:
            stream = t.cuda.current_stream(idx)
        key = (idx, stream.cuda_stream)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                with t.cuda.device(idx), t.cuda.stream(stream):
                    buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=dev)
                self._bufs[key] = buf
            return buf

    def clear(self):
        with self._lock:
            self._bufs.clear()


class SortOverflowError(RuntimeError):
    """The device reported dropped work (bs_sort_status != 0): the output is not sorted."""


def check_status(status) -> None:
    """Raise if a device status word (CUDA int32[1] filled by bs_sort_status) is set (syncs)."""
    v = int(status.item())
    if v:
        what = [n for b, n in ((1, "bucket list"), (2, "tile map"), (4, "task list"),
                               (8, "debug-build bounds check")) if v & b]
        raise SortOverflowError(f"device work-list overflow ({', '.join(what)}; status {v}): output is not sorted")


workspaces = _WorkspaceCache()


def sort_words_device(keys, vals=None, *, width: int, start_pos: int = 0, key_kind: int = 0,
                      counters=None, depth: int = 1, workspace=None, check: bool = True):
    """Sort a contiguous 1-D CUDA tensor of raw words in place (bs_sort).

    ``counters``: optional CUDA int64[4] tensor receiving the reference Metrics.
    ``workspace``: optional CUDA uint8 tensor (defaults to the (device, stream) cache).
    ``check``: read the device overflow status back and raise
    :class:`SortOverflowError` if work was dropped (one stream sync).  With
    ``check=False`` the status tensor is returned for a deferred
    :func:`check_status` (the timed bench loop).
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
        if n <= 1 or width - start_pos <= 0:
            return None  # nothing launched
        # the sort's status word, read in place from the workspace (no copy
        # launched); valid until the workspace's next sort
        off = int(L.bs_sort_status_offset())
        status = workspace[off:off + 4].view(t.int32)
    if check:
        check_status(status)
        return None
    return status


def exact_sort_device(keys, vals=None, *, width: int, start_pos: int = 0, key_kind: int = 0,
                      mode: int = _lib.EX_REC, passthrough_loop: bool = False, check_after: int = 0,
                      streak: int = 0, checked: bool = False, par_levels: int = 0, depth: int = 1,
                      counters=None, on_level=None):
    """Reference-order sort of a contiguous 1-D CUDA word tensor in place (bs_exact_sort).

    ``mode``: ``_lib.EX_REC`` (kernels.sort_words with its switches),
    ``EX_ITER`` (sort_words_iterative), ``EX_LEVELS`` (the level observer
    engine, core._sort_levels) or ``EX_PAR`` (sort_parallel with
    ``par_levels`` prepartition levels).  ``counters``: CUDA int64[4] that
    receives the reference counters (overwritten).  ``on_level(pos, starts, current)``: called after every level with the
    segment start positions (numpy uint32, ascending) and the array's current
    contents (a CUDA word tensor) -- syncs the stream once per level.
    """
    t = require_cuda()
    if not keys.is_cuda or keys.dim() != 1 or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous 1-D CUDA tensor")
    n = keys.numel()
    kb = keys.element_size()
    vb, vptr = 0, None
    if vals is not None:
        if not vals.is_cuda or vals.dim() != 1 or not vals.is_contiguous() or vals.numel() != n:
            raise ValueError("values must be a contiguous 1-D CUDA tensor of the same length")
        vb, vptr = vals.element_size(), vals.data_ptr()
    if counters is not None and (counters.dtype != t.int64 or counters.numel() != 4 or not counters.is_cuda):
        raise ValueError("counters must be a CUDA int64[4] tensor")
    L = _lib.lib()
    ws = workspaces.get(L.bs_exact_workspace_bytes(n, kb, vb), keys.device)
    sptr = stream_ptr(keys.device)
    cb = None
    errors = []
    if on_level is not None:
        starts = t.empty(max(1, n), dtype=t.int32, device=keys.device)
        cnt = t.zeros(1, dtype=t.int32, device=keys.device)
        snap = t.empty_like(keys)

        def _level(_ctx, pos):
            try:
                _lib.check(L.bs_exact_boundaries(ws.data_ptr(), n, kb, vb, starts.data_ptr(), cnt.data_ptr(), sptr))
                _lib.check(L.bs_exact_snapshot(keys.data_ptr(), ws.data_ptr(), n, kb, vb, int(pos) - int(start_pos) + 1,
                                               snap.data_ptr(), sptr))
                m = int(cnt.item())
                on_level(int(pos), starts[:m].cpu().numpy().view(np.uint32), snap)
            except BaseException as e:  # raised again after the C call returns
                errors.append(e)

        cb = _lib.LEVEL_FN(_level)
    with t.cuda.device(keys.device):
        rc = L.bs_exact_sort(keys.data_ptr(), vptr, n, kb, vb, int(width), int(start_pos), int(key_kind), int(mode),
                             int(bool(passthrough_loop)), int(check_after), int(streak), int(bool(checked)),
                             int(par_levels), int(depth), ws.data_ptr(), ws.numel(), sptr,
                             counters.data_ptr() if counters is not None else None,
                             cb if cb is not None else _lib.LEVEL_FN(), None)
    _lib.check(rc)
    if errors:
        raise errors[0]


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
