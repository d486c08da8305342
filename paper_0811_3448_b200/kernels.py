"""The reference kernel-module ABI (``binarsort.kernels``) on sm_100a CUDA.

Reference: ``/root/reference/pkg/src/binarsort/kernels.py``.  Same function
names, argument meanings and counter layout (int64[4] = extractions, swaps,
calls, max depth; kernels.py:9-17), so callers written against the numba
module (core/variants/tests) run unchanged.  ``arr`` may be a 1-D numpy word
array (copied to the device and back) or a CUDA tensor (sorted in place).
``counters`` may be a numpy int64[4] (host) or a CUDA int64 tensor.

Backend selection mirrors kernels.py:19-35: ``BINARSORT_BACKEND`` must be
``auto`` or ``cuda``; anything else raises ``ValueError`` at import.  There
is no CPU fallback.

Counter exactness: every entry point returns the reference's counters
exactly.  ``partition_words`` uses the closed form of the two-cursor loop
(SURVEY Appendix A).  ``sort_words`` with the baseline switches on a
full-width word range runs the fast digit sort and the closed-form counters
(Appendix B); every other case -- the optimisation switches, a start bit
``pos > 0`` or words wider than ``width`` (where the order of equal keys
shows), and ``sort_words_iterative`` (stack high-water mark) -- runs the exact
reference-order engine (``bs_exact_sort``, exact_impl.cuh), which replays the
recursion's partitions level by level.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib, device

EXTRACTIONS, SWAPS, CALLS, MAX_DEPTH = 0, 1, 2, 3

_choice = os.environ.get("BINARSORT_BACKEND", "auto").strip().lower() or "auto"
if _choice not in ("auto", "cuda"):
    raise ValueError(f"BINARSORT_BACKEND must be 'auto' or 'cuda' for the B200 backend, got {_choice!r}")

BACKEND = "cuda"


def new_counters() -> np.ndarray:
    return np.zeros(4, dtype=np.int64)


class _Range:
    """Device view of arr[lower..upper] with write-back for host arrays."""

    def __init__(self, arr, lower, upper):
        t = device.require_cuda()
        self.arr, self.lower, self.upper = arr, int(lower), int(upper)
        if device.is_torch_tensor(arr):
            view = arr[self.lower:self.upper + 1]
            if view.is_cuda and view.is_contiguous():
                self.dev = device.as_raw_words(view)
                self._host = None
            else:
                self.dev = device.as_raw_words(view.to("cuda").contiguous())
                self._host = view
        else:
            if not isinstance(arr, np.ndarray) or arr.ndim != 1 or arr.dtype.kind not in "ui":
                raise TypeError("kernels operate on 1-D unsigned word arrays")
            view = arr[self.lower:self.upper + 1]
            self.dev = device.to_device_words(view)
            self._host = view
        self.t = t

    def commit(self):
        if self._host is None:
            return
        if isinstance(self._host, np.ndarray):
            self._host[...] = self.dev.cpu().numpy().view(self._host.dtype)
        else:
            self._host.copy_(self.dev.view(self._host.dtype).to(self._host.device))


def _counter_tensor(counters, t, dev):
    c = t.zeros(4, dtype=t.int64, device=dev)
    return c


def _merge_counters(counters, c_dev, *, add_depth_max=True):
    c = c_dev.cpu().numpy()
    if device.is_torch_tensor(counters):
        host = counters.cpu().numpy()
        host[:3] += c[:3]
        host[3] = max(host[3], c[3])
        counters.copy_(device.torch().from_numpy(host))
    else:
        counters[:3] += c[:3]
        counters[3] = max(int(counters[3]), int(c[3]))


def partition_words(arr, lower, upper, pos, width, counters) -> int:
    """One two-cursor partition pass on arr[lower..upper] at bit pos (kernels.py:56-77).

    Exact reference permutation and split; bumps counters[0] by the range size
    and counters[1] by the swap count.  Returns ``upper + 1`` when every bit is 0.
    """
    if upper < lower:
        return int(lower)
    r = _Range(arr, lower, upper)
    c = r.t.zeros(4, dtype=r.t.int64, device=r.dev.device)
    split = device.partition_device(r.dev, width=width, pos=pos, counters=c)
    r.commit()
    _merge_counters(counters, c)
    return int(lower) + int(split.item())


def range_sorted_words(arr, lower, upper) -> bool:
    """arr[lower..upper] nondecreasing as unsigned words (kernels.py:80-85)."""
    if upper <= lower:
        return True
    r = _Range(arr, lower, upper)
    return device.range_sorted_device(r.dev)


def sort_words(arr, lower, upper, pos, width, passthrough_loop, check_after, streak, checked,
               counters, depth) -> None:
    """Sort arr[lower..upper] by bits pos..width-1 (kernels.py:88-126)."""
    n = int(upper) - int(lower) + 1
    if n < 2 or pos >= width:
        # base case: one call at this depth (kernels.py:100-105)
        _bump_call(counters, depth)
        return
    r = _Range(arr, lower, upper)
    c = r.t.zeros(4, dtype=r.t.int64, device=r.dev.device)
    baseline = not passthrough_loop and int(check_after) == 0
    if baseline and int(pos) == 0 and r.dev.element_size() * 8 == int(width):
        device.sort_words_device(r.dev, width=width, start_pos=pos, key_kind=_lib.BS_KEY_UNSIGNED,
                                 counters=c, depth=depth)
    else:
        device.exact_sort_device(r.dev, width=width, start_pos=pos, key_kind=_lib.BS_KEY_UNSIGNED,
                                 mode=_lib.EX_REC, passthrough_loop=bool(passthrough_loop),
                                 check_after=int(check_after), streak=int(streak), checked=bool(checked),
                                 depth=int(depth), counters=c)
    r.commit()
    _merge_counters(counters, c)


def sort_words_iterative(arr, lower, upper, width, counters) -> None:
    """Explicit-stack form (kernels.py:129-172): calls = partitions, max_depth = stack high-water."""
    n = int(upper) - int(lower) + 1
    if n < 1:
        # an empty range is pushed once and passes through every bit (kernels.py:138-160)
        _bump_calls(counters, int(width), 1)
        return
    r = _Range(arr, lower, upper)
    c = r.t.zeros(4, dtype=r.t.int64, device=r.dev.device)
    device.exact_sort_device(r.dev, width=width, start_pos=0, key_kind=_lib.BS_KEY_UNSIGNED,
                             mode=_lib.EX_ITER, counters=c)
    r.commit()
    _merge_counters(counters, c)


def _bump_calls(counters, calls, depth):
    if device.is_torch_tensor(counters):
        host = counters.cpu().numpy()
        host[CALLS] += calls
        host[MAX_DEPTH] = max(int(host[MAX_DEPTH]), int(depth))
        counters.copy_(device.torch().from_numpy(host))
    else:
        counters[CALLS] += calls
        counters[MAX_DEPTH] = max(int(counters[MAX_DEPTH]), int(depth))


def _bump_call(counters, depth):
    if device.is_torch_tensor(counters):
        host = counters.cpu().numpy()
        host[CALLS] += 1
        host[MAX_DEPTH] = max(int(host[MAX_DEPTH]), int(depth))
        counters.copy_(device.torch().from_numpy(host))
    else:
        counters[CALLS] += 1
        counters[MAX_DEPTH] = max(int(counters[MAX_DEPTH]), int(depth))
