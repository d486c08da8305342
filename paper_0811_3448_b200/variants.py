"""Iterative / optimized / parallel drive forms (drop-in for ``binarsort.variants``).

Reference: ``/root/reference/pkg/src/binarsort/variants.py``.  All three
produce element-for-element the reference's output AND its counters:

* ``sort_iterative`` -- explicit work stack (variants.py:67-90): calls count
  partitions, ``max_depth`` is the stack high-water mark;
* ``sort_optimized`` -- pass-through loop (no call, no depth) and the
  sortedness scan after a streak of pass-throughs (variants.py:93-121), which
  inspects the range's current, partially partitioned content;
* ``sort_parallel`` -- ``ceil(lg workers)`` levels of level-synchronous
  prepartition, then one recursive sort per bucket from that bit
  (variants.py:124-229).

On the device they run as modes of the exact reference-order engine
(``bs_exact_sort``, exact_impl.cuh): every reference call works on a disjoint
index range, so replaying all ranges of one bit level together reproduces the
reference's array states, and with them the counters.  The thread pool of
``sort_parallel`` has no device counterpart -- every bucket of a level is
processed concurrently by all SMs.  Inputs whose counters need no replay
(``sort_optimized`` with both switches off) take the fast digit sort;
multi-GPU sharding is ``paper_0811_3448_b200.dist``.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib, core
from .core import Metrics

__all__ = ["OptimizationConfig", "sort_iterative", "sort_optimized", "sort_parallel"]


@dataclass
class OptimizationConfig:
    """Pass-through shortcuts (variants.py:17-33)."""

    passthrough_loop: bool = True
    sortedness_check_after: int = 4

    def __post_init__(self):
        if self.sortedness_check_after < 0:
            raise ValueError("sortedness_check_after must be >= 0")


def _finish(out: Metrics, provided: Metrics | None) -> Metrics:
    if provided is not None:
        provided.merge(out)
        return provided
    return out


def _run(seq, codec, **kw) -> Metrics:
    out = Metrics()
    n = len(seq)
    if n <= 1:
        return out
    width = codec.width_for(seq)
    if width == 0:
        return out
    core._sort_device(seq, codec, None, width, 0, 1, out, **kw)
    return out


def sort_iterative(seq, codec, metrics: Metrics | None = None) -> Metrics:
    """Explicit work-stack sort (variants.py:67-90); max_depth = stack high-water mark."""
    return _finish(_run(seq, codec, mode=_lib.EX_ITER), metrics)


def sort_optimized(seq, codec, config: OptimizationConfig | None = None,
                   metrics: Metrics | None = None) -> Metrics:
    """Pass-through loop and sortedness-scan shortcuts (variants.py:93-121).

    With both switches off this is the recursive baseline, counters included.
    """
    if config is None:
        config = OptimizationConfig()
    if not config.passthrough_loop and config.sortedness_check_after == 0:
        return _finish(_run(seq, codec), metrics)
    return _finish(_run(seq, codec, mode=_lib.EX_REC, passthrough_loop=config.passthrough_loop,
                        check_after=config.sortedness_check_after), metrics)


def sort_parallel(seq, codec, workers: int, metrics: Metrics | None = None) -> Metrics:
    """Bucket-parallel sort (variants.py:162-229); ``workers`` must be >= 1.

    ``levels = min(ceil(lg workers), width)`` prepartition levels, then the
    recursive sort of every bucket from bit ``levels`` at depth ``levels + 1``
    -- the reference's partitions and counters.
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    n = len(seq)
    if n <= 1:
        return _finish(Metrics(), metrics)
    width = codec.width_for(seq)
    if width == 0:
        return _finish(Metrics(), metrics)
    levels = min((workers - 1).bit_length(), width)
    return _finish(_run(seq, codec, mode=_lib.EX_PAR, par_levels=levels), metrics)
