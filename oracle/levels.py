"""Level-synchronous observer engine -- TEST INFRASTRUCTURE ONLY.

Restates the reference's ``core._sort_levels`` (core.py:146-180) over a word
array, using the oracle's ``partition_words`` (kernels.py:56-77 restated in
C) and ``range_sorted_words`` (kernels.py:80-85): before each partition the
range is scanned for sortedness (a sorted range stops), one call is counted
per partition, and the observer receives ``(pos, [(lo, up), ...])`` after
every bit level.  Pinned against the reference's traces in
tests/golden/golden_variants.json (tests/test_oracle_golden.py).
"""

from __future__ import annotations

from . import new_counters, partition_words, range_sorted_words


def sort_levels(arr, lower: int, upper: int, start_pos: int, width: int, observer):
    """Returns counters [extractions, swaps, calls, max_depth]."""
    c = new_counters()
    calls = 0
    max_depth = 0
    segments = [(lower, upper, upper > lower)]
    for pos in range(start_pos, width):
        nxt = []
        worked = False
        for lo, up, active in segments:
            if not active:
                nxt.append((lo, up, False))
                continue
            if range_sorted_words(arr, lo, up):
                nxt.append((lo, up, False))
                continue
            worked = True
            calls += 1
            split = partition_words(arr, lo, up, pos, width, c)
            if split == lo or split == up + 1:
                nxt.append((lo, up, True))
            else:
                nxt.append((lo, split - 1, split - 1 > lo))
                nxt.append((split, up, up > split))
        segments = nxt
        if worked and pos + 1 - start_pos > max_depth:
            max_depth = pos + 1 - start_pos
        observer(pos, [(lo, up) for lo, up, _ in segments])
    c[2] += calls
    c[3] = max(int(c[3]), max_depth)
    return c
