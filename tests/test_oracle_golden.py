"""Pin the CPU oracle (oracle/binarsort_oracle.c) to the reference's own outputs.

tests/golden/golden.json was produced by running the reference package
(tests/golden/make_golden.py).  These tests only use the oracle (the checker),
never the product; they need no GPU.
"""

import hashlib

import numpy as np
import pytest

from paper_0811_3448_b200.cases import config1


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_nybble_worked_example(oracle_lib, golden):
    # PAPER.md:300-316; reference tests/test_core.py:105-110
    g = golden["nybble_sort"]
    a = np.array(g["input"], dtype=np.uint32)
    c = oracle_lib.sort(a, 4)
    assert a.tolist() == g["output"] == [0, 0, 4, 7, 10, 11, 12, 14]
    assert c.tolist() == g["metrics"] == [28, 13, 16, 5]


def test_paper_partitions(oracle_lib, golden):
    # tests/test_core.py:33-63 and tests/test_kernels.py:45-52
    for p in golden["partitions_w4"]:
        a = np.array(p["input"], dtype=np.uint32)
        c = oracle_lib.new_counters()
        split = oracle_lib.partition_words(a, 0, a.size - 1, p["pos"], 4, c)
        assert a.tolist() == p["output"]
        assert split == p["split"]
        assert c[0] == p["extractions"] and c[1] == p["swaps"]


def test_zero_one_depth(oracle_lib, golden):
    # tests/test_core.py:160-164: [0, 1] at width 8 -> depth 9
    a = np.array([0, 1], dtype=np.uint32)
    assert oracle_lib.sort(a, 8).tolist() == golden["zero_one_w8"]
    assert golden["zero_one_w8"][3] == 9


def test_kernel_sorts_match_reference(oracle_lib, golden):
    # tests/test_kernels.py:34-42 sizes, counters included
    rng = {32: np.random.default_rng(21), 64: np.random.default_rng(21)}
    for g in golden["kernel_sorts"]:
        w, size = g["width"], g["size"]
        dt = np.uint32 if w == 32 else np.uint64
        v = rng[w].integers(0, 2 ** w, size, dtype=np.uint64).astype(dt)
        assert sha(v) == g["input_sha"]
        a = v.copy()
        c = oracle_lib.new_counters()
        if size > 1:
            oracle_lib.sort_words(a, 0, size - 1, 0, w, False, 0, 0, False, c, 1)
        assert sha(a) == g["output_sha"], (w, size)
        assert c.tolist() == g["counters"], (w, size)


def test_kernel_partitions_match_reference(oracle_lib, golden):
    rng = np.random.default_rng(5)
    for g in golden["kernel_partitions"]["cases"]:
        n = int(rng.integers(1, 3000))
        w = int(rng.choice([8, 16, 32]))
        pos = int(rng.integers(0, w))
        v = rng.integers(0, 2 ** w, n, dtype=np.uint64).astype(np.uint32)
        assert (n, w, pos) == (g["n"], g["width"], g["pos"]) and sha(v) == g["input_sha"]
        a = v.copy()
        c = oracle_lib.new_counters()
        split = oracle_lib.partition_words(a, 0, n - 1, pos, w, c)
        assert sha(a) == g["output_sha"] and split == g["split"] and c.tolist() == g["counters"]


def test_cfg1_matches_reference(oracle_lib, golden):
    # BASELINE.json configs[0]: 2^20 u32 from seed 0, sorted by the reference
    g = golden["cfg1"]
    x = config1()
    assert sha(x) == g["input_sha"]
    a = x.copy()
    c = oracle_lib.sort(a, 32)
    assert sha(a) == g["output_sha"]
    assert c.tolist() == g["metrics"]


def test_iterative_and_parallel_restatements(oracle_lib):
    # kernels.py:129-172 and variants.py:162-229: identical output
    rng = np.random.default_rng(22)
    for size in (2, 50, 700, 5000):
        base = rng.integers(0, 2 ** 32, size, dtype=np.uint64).astype(np.uint32)
        a, b, p = base.copy(), base.copy(), base.copy()
        ca, cb = oracle_lib.sort(a, 32), oracle_lib.new_counters()
        oracle_lib.sort_words_iterative(b, 0, size - 1, 32, cb)
        assert np.array_equal(a, b) and ca[0] == cb[0] and ca[1] == cb[1] and cb[3] <= 33
        for workers in (1, 2, 3, 8):
            q = base.copy()
            m = oracle_lib.sort_parallel(q, workers)
            assert np.array_equal(q, a)
            assert m[0] == ca[0] and m[1] == ca[1]
        assert np.array_equal(p[np.argsort(p, kind="stable")], a)


def test_sortedness_check_lowers_extractions(oracle_lib):
    # tests/test_kernels.py:70-75
    arr = np.arange(5000, dtype=np.uint32)
    fast, slow = oracle_lib.new_counters(), oracle_lib.new_counters()
    oracle_lib.sort_words(arr.copy(), 0, arr.size - 1, 0, 32, True, 1, 0, False, fast, 1)
    oracle_lib.sort_words(arr.copy(), 0, arr.size - 1, 0, 32, False, 0, 0, False, slow, 1)
    assert fast[0] < slow[0]


def test_parallel_zero_workers_rejected(oracle_lib):
    with pytest.raises(ValueError):
        oracle_lib.sort_parallel(np.array([2, 1], dtype=np.uint32), 0)
