"""The sort entry points (drop-in for ``binarsort.core``), backed by sm_100a CUDA.

Reference: ``/root/reference/pkg/src/binarsort/core.py``.  ``sort`` keeps the
reference signature ``sort(seq, codec) -> Metrics`` (core.py:201-222): the
sequence is sorted in place and the reference's work counters are returned.
Where the reference hands a word array to ``kernels.sort_words``
(core.py:213-219), this module hands the device words to ``bs_sort`` in
``libbinarsort_b200.so``; the counters come from the closed form over the
sorted output, computed on the GPU.

Accepted sequences: 1-D numpy arrays (any stride), 1-D torch tensors (CUDA
ones are sorted in place on their device), and lists/tuples of ints or floats
for the word codecs.  Element types only the reference's generic Python
engine can sort (byte strings, custom tuple codecs) raise ``TypeError``:
that engine is not part of the B200 hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, device
from .device import is_torch_tensor

EXTRACTIONS, SWAPS, CALLS, MAX_DEPTH = 0, 1, 2, 3


@dataclass
class SortRange:
    """Inclusive bounds plus the current bit position, 0 = MSB (core.py:21-35)."""

    lower: int
    upper: int
    pos: int = 0

    def __post_init__(self):
        assert self.lower >= 0, "lower bound must be >= 0"
        assert self.upper >= self.lower - 1, "upper may be at most one below lower"
        assert self.pos >= 0, "bit position must be >= 0"

    def is_empty(self) -> bool:
        return self.upper < self.lower


@dataclass
class PartitionResult:
    """``split`` = first index of the bit-1 side; ``pass_through`` = one side empty (core.py:38-48)."""

    split: int
    pass_through: bool


@dataclass
class Metrics:
    """Reference work counters (core.py:51-77)."""

    bit_extractions: int = 0
    swaps: int = 0
    recursive_calls: int = 0
    max_depth: int = 0

    def merge(self, other: "Metrics") -> None:
        """Counts add, depth takes the max (core.py:60-70)."""
        self.bit_extractions += other.bit_extractions
        self.swaps += other.swaps
        self.recursive_calls += other.recursive_calls
        self.max_depth = max(self.max_depth, other.max_depth)

    def _add_counters(self, counters) -> None:
        c = [int(v) for v in counters]
        self.merge(Metrics(c[EXTRACTIONS], c[SWAPS], c[CALLS], c[MAX_DEPTH]))


# ---------------------------------------------------------------------------
# sequence <-> device words
# ---------------------------------------------------------------------------

class DeviceWords:
    """Contiguous raw-word CUDA tensor(s) for a sequence, with write-back.

    ``keys`` is an int32/int64 CUDA tensor holding the caller's raw words
    (the codec transform is applied on the device, not here).
    """

    def __init__(self, seq, codec, values=None, lower: int = 0, upper: int | None = None):
        kind = codec.gpu_spec(seq)
        if kind is None:
            raise TypeError(
                f"{type(codec).__name__} on {type(seq).__name__} has no word view; the B200 backend "
                "sorts 1-D integer/float arrays, tensors and lists only (generic engine is out of scope)")
        self.seq = seq
        self.key_kind = kind
        self.lower = lower
        self.upper = (len(seq) - 1) if upper is None else upper
        self._vals_src = values
        t = device.require_cuda()
        self._writeback = None
        self.keys = self._upload(seq, t, is_key=True, codec=codec)
        self.vals = None
        if values is not None:
            if len(values) != len(seq):
                raise ValueError("values must have the same length as the keys")
            self.vals = self._upload(values, t, is_key=False, codec=None)

    # ---- upload ---------------------------------------------------------
    def _upload(self, seq, t, *, is_key, codec):
        lo, hi = self.lower, self.upper + 1
        want_float = is_key and self.key_kind == _lib.BS_KEY_FLOAT
        if is_torch_tensor(seq):
            view = seq[lo:hi]
            src = view
            if want_float and view.dtype != t.float64:
                src = view.to(t.float64)
            elif view.element_size() not in (4, 8):
                src = view.to(t.float64 if view.dtype.is_floating_point else t.int64)
            if src is view and view.is_cuda and view.is_contiguous():
                return device.as_raw_words(view)  # sorted in place on its device
            dev = device.as_raw_words(src.to("cuda").contiguous())
            src_dtype = src.dtype

            def wb(cur=None):
                res = (dev if cur is None else cur).view(src_dtype)
                view.copy_(res if res.dtype == view.dtype else res.to(view.dtype))  # D2H straight into view

            self._chain(wb)
            return dev
        if isinstance(seq, np.ndarray):
            view = seq[lo:hi]
            if not view.flags.writeable:
                raise ValueError("cannot sort a read-only array in place")
            if want_float and view.dtype != np.float64:
                host = view.astype(np.float64)
            elif view.dtype.itemsize not in (4, 8):
                host = view.astype(np.float64 if view.dtype.kind == "f" else np.int64)
            else:
                host = view
            dev = device.to_device_words(host)
            host_dtype = host.dtype

            def wb(cur=None):
                out = (dev if cur is None else cur).cpu().numpy().view(host_dtype)
                view[...] = out if out.dtype == view.dtype else out.astype(view.dtype)

            self._chain(wb)
            return dev
        if isinstance(seq, list):
            items = seq[lo:hi]
            if want_float:
                host = np.asarray(items, dtype=np.float64)
            else:
                if any(not isinstance(v, (int, np.integer)) for v in items):
                    raise TypeError("list keys must be ints for an integer codec")
                host = np.array([int(v) & 0xFFFFFFFFFFFFFFFF for v in items], dtype=np.uint64)
            negative = (not want_float) and any(int(v) < 0 for v in items)
            dev = device.to_device_words(host)

            def wb(cur=None):
                out = (dev if cur is None else cur).cpu().numpy().view(host.dtype)
                if want_float:
                    seq[lo:hi] = [float(v) for v in out]
                elif negative:
                    seq[lo:hi] = [int(v) for v in out.view(np.int64)]
                else:
                    seq[lo:hi] = [int(v) for v in out]

            self._chain(wb)
            return dev
        raise TypeError(f"unsupported sequence type {type(seq).__name__} (tuples are immutable)")

    def _chain(self, fn):
        prev = self._writeback
        if prev is None:  # the first writeback is the keys'
            self._writeback = self._key_wb = fn
            return

        def both():
            prev()
            fn()

        self._writeback = both

    def commit(self):
        if self._writeback is not None:
            self._writeback()

    def show_keys(self, current) -> None:
        """Write a device word tensor (the keys' current state) into the caller's sequence.

        A CUDA tensor sorted in place needs nothing: its storage is not the
        engine's ping-pong state, so it is written from ``current`` too."""
        wb = getattr(self, "_key_wb", None)
        if wb is not None:
            wb(current)
        else:
            self.keys.copy_(current)


# ---------------------------------------------------------------------------
# public entry points
# ---------------------------------------------------------------------------

def partition(seq, rng: SortRange, codec, metrics: Metrics, values=None) -> PartitionResult:
    """One reference partition pass on ``seq[rng.lower..rng.upper]`` at bit ``rng.pos``.

    Same contract as core.partition (core.py:94-107), including the exact
    unstable two-cursor permutation of ``_partition_span`` (core.py:80-91),
    reproduced on the GPU by its closed form.  ``values``
    (extension) receives the same permutation, which is how the reference's
    tagged-element test (tests/test_core.py:65-71) is expressed for words.
    """
    width = codec.width_for(seq)
    assert not rng.is_empty(), "partition requires a non-empty range"
    assert rng.upper < len(seq), "range exceeds sequence bounds"
    assert 0 <= rng.pos < width, "bit position out of codec width"
    t = device.require_cuda()
    w = DeviceWords(seq, codec, values, lower=rng.lower, upper=rng.upper)
    counters = t.zeros(4, dtype=t.int64, device=w.keys.device)
    enc = _Encoder(w, width)
    enc.apply()
    split = device.partition_device(w.keys, w.vals, width=width, pos=rng.pos, counters=counters)
    enc.undo()
    w.commit()
    c = counters.cpu().numpy()
    metrics.bit_extractions += int(c[EXTRACTIONS])
    metrics.swaps += int(c[SWAPS])
    s = rng.lower + int(split.item())
    return PartitionResult(s, s == rng.lower or s == rng.upper + 1)


class _Encoder:
    """In-place device codec transform for the partition pass (which reads raw bits).

    The reference's ``partition`` reads bits through ``codec.bit_at`` (the
    encoded key, keys.py:191-193,216-218); the partition kernel reads raw
    words, so signed/float words are encoded on the device before the pass and
    decoded after it.  Sorting never needs this (the sort kernels fuse it).
    """

    def __init__(self, w, width):
        self.w, self.width = w, width

    def _flip(self):
        t = device.torch()
        k = self.w.keys
        bits = k.element_size() * 8
        v = 1 << (bits - 1) if self.w.key_kind == _lib.BS_KEY_FLOAT else 1 << (self.width - 1)
        return t.tensor(v - (1 << bits) if v >> (bits - 1) else v, dtype=k.dtype, device=k.device)

    def apply(self):
        k = self.w.keys
        if self.w.key_kind == _lib.BS_KEY_SIGNED:
            k ^= self._flip()
        elif self.w.key_kind == _lib.BS_KEY_FLOAT:
            t = device.torch()
            k.copy_(t.where(k < 0, ~k, k | self._flip()))

    def undo(self):
        k = self.w.keys
        if self.w.key_kind == _lib.BS_KEY_SIGNED:
            k ^= self._flip()
        elif self.w.key_kind == _lib.BS_KEY_FLOAT:
            t = device.torch()
            k.copy_(t.where(k < 0, k ^ self._flip(), ~k))


def binar_sort_range(seq, rng: SortRange, codec, metrics: Metrics, observer=None) -> None:
    """Sort ``seq[rng.lower..rng.upper]`` in place from bit ``rng.pos`` (core.py:183-198).

    With an ``observer`` the level-synchronous engine runs and reports the
    sub-array boundaries after every bit level (core.py:146-180), exactly as
    the reference's does (same partitions, same sortedness stops, same
    counters).
    """
    assert rng.is_empty() or (rng.lower >= 0 and rng.upper < len(seq)), "range exceeds sequence bounds"
    if rng.is_empty():
        return
    width = codec.width_for(seq)
    assert rng.pos <= width, "bit position past codec width"
    if observer is not None:
        _sort_levels_device(seq, codec, width, rng.lower, rng.upper, rng.pos, metrics, observer)
        return
    n = rng.upper - rng.lower + 1
    if n < 2 or rng.pos == width:
        # the reference's base case still counts one call at depth 1 (kernels.py:100-105)
        metrics.recursive_calls += 1
        metrics.max_depth = max(metrics.max_depth, 1)
        return
    _sort_device(seq, codec, None, width, rng.pos, 1, metrics, rng.lower, rng.upper)


def _word_bits(w) -> int:
    return w.keys.element_size() * 8


def _tie_order_observable(w, width: int, start_pos: int) -> bool:
    """Could two words equal in the examined key bits differ elsewhere?

    Only then does the order among equal keys show in a keys-only result; the
    fast sort (unique nondecreasing output) is bit-exact otherwise.
    """
    return start_pos > 0 or width < _word_bits(w)


def _sort_device(seq, codec, values, width, start_pos, depth, metrics, lower=0, upper=None,
                 with_metrics=True, exact=None, mode=None, _holder=None, **exact_kw):
    if codec.gpu_spec(seq) is None:  # generic-engine element types: out of scope
        raise TypeError(f"{type(codec).__name__} on {type(seq).__name__} has no word view "
                        "(the B200 backend sorts 1-D integer/float arrays, tensors and lists)")
    t = device.require_cuda()
    w = DeviceWords(seq, codec, values, lower=lower, upper=upper)
    if _holder is not None:
        _holder["w"] = w
    counters = t.zeros(4, dtype=t.int64, device=w.keys.device) if with_metrics else None
    if exact is None:
        exact = mode is not None or (values is None and _tie_order_observable(w, width, start_pos))
    if exact:
        device.exact_sort_device(w.keys, w.vals, width=width, start_pos=start_pos, key_kind=w.key_kind,
                                 mode=_lib.EX_REC if mode is None else mode, depth=depth, counters=counters,
                                 **exact_kw)
    else:
        device.sort_words_device(w.keys, w.vals, width=width, start_pos=start_pos, key_kind=w.key_kind,
                                 counters=counters, depth=depth)
    w.commit()
    if with_metrics and metrics is not None:
        metrics._add_counters(counters.cpu().numpy())


def _sort_levels_device(seq, codec, width, lower, upper, start_pos, metrics, observer):
    """core._sort_levels (core.py:146-180) on the device: the observer sees (pos, [(lo, up), ...])."""
    n = upper - lower + 1

    holder = {}

    def on_level(pos, starts, current):
        w = holder.get("w")
        if w is not None:  # the observer reads the partially sorted sequence (core.py:175-180)
            w.show_keys(current)
        ends = np.empty(len(starts), dtype=np.int64)
        ends[:-1] = starts[1:].astype(np.int64) - 1
        if len(starts):
            ends[-1] = n - 1
        observer(pos, [(lower + int(a), lower + int(b)) for a, b in zip(starts, ends)])

    if start_pos >= width:
        return
    if n < 2:  # segments = [(lower, upper, False)]: no work, the observer still sees every level
        for pos in range(start_pos, width):
            observer(pos, [(lower, upper)])
        return
    _sort_device(seq, codec, None, width, start_pos, 1, metrics, lower, upper, mode=_lib.EX_LEVELS,
                 on_level=on_level, _holder=holder)


def sort(seq, codec, values=None, *, with_metrics: bool = True, exact: bool | None = None) -> Metrics:
    """Sort ``seq`` in place into nondecreasing codec order; return Metrics (core.py:201-222).

    ``values`` (extension): a same-length sequence permuted alongside the
    keys.  By default the device sort is stable, so equal keys keep their
    input order and every value stays with its key.

    ``exact``: ``None`` (default) picks the fast digit sort whenever the
    order of equal keys cannot be observed (keys only, full-width words) and
    the exact reference-order engine otherwise (``UnsignedCodec(w)`` on wider
    words, lists); ``True`` always replays the reference's own (unstable)
    permutations -- also for ``values``; ``False`` always takes the fast sort.
    """
    metrics = Metrics()
    n = len(seq)
    if n <= 1:
        return metrics
    width = codec.width_for(seq)
    if width == 0:
        return metrics
    _sort_device(seq, codec, values, width, 0, 1, metrics, with_metrics=with_metrics, exact=exact)
    return metrics


def sort_with_observer(seq, codec, observer) -> Metrics:
    """Sort ``seq`` while reporting sub-array boundaries per bit level (core.py:225-239).

    The observer is called once per bit position with ``(pos, boundaries)``.
    Inputs of fewer than two elements sort trivially with no callbacks.
    """
    metrics = Metrics()
    n = len(seq)
    if n <= 1:
        return metrics
    width = codec.width_for(seq)
    if width == 0:
        return metrics
    _sort_levels_device(seq, codec, width, 0, n - 1, 0, metrics, observer)
    return metrics
