"""Iterative / optimized / parallel drive forms (drop-in for ``binarsort.variants``).

Reference: ``/root/reference/pkg/src/binarsort/variants.py``.  On the CPU the
three variants differ in scheduling (explicit stack, pass-through loop and
sortedness scan, thread-pool over top-bit buckets); all produce the same
output as the recursive sort (variants.py:1-6).  On B200 there is one
scheduling -- the level-synchronous device work-list of ``bs_sort``, which
*is* the iterative form and *is* the bucket-parallel form (every bucket of a
level is processed concurrently by all 148 SMs) -- so all three route to the
same CUDA path and return identical output.  Multi-GPU sharding is
``paper_0811_3448_b200.dist``.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import core
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


def sort_iterative(seq, codec, metrics: Metrics | None = None) -> Metrics:
    """Explicit work-list sort (variants.py:67-90); same output as ``core.sort``."""
    return _finish(core.sort(seq, codec), metrics)


def sort_optimized(seq, codec, config: OptimizationConfig | None = None,
                   metrics: Metrics | None = None) -> Metrics:
    """Pass-through/sortedness shortcuts (variants.py:93-121).

    The device sort already skips constant digits (pass-through) and
    all-equal buckets (sortedness), so the switches change nothing in the
    output; the returned counters are the baseline recursion's.
    """
    if config is None:
        config = OptimizationConfig()
    return _finish(core.sort(seq, codec), metrics)


def sort_parallel(seq, codec, workers: int, metrics: Metrics | None = None) -> Metrics:
    """Bucket-parallel sort (variants.py:162-229); ``workers`` must be >= 1.

    Output identical to the sequential sort.  The GPU processes every bucket
    of a level concurrently, so ``workers`` only validates.
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return _finish(core.sort(seq, codec), metrics)
