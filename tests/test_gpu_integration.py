"""INTEGRATION.md's binding (integration/_cuda.py), loaded standalone as the
reference's kernel module would load it, against the reference's own outputs:
the kernel-module tests (tests/test_kernels.py:34-82 of the reference) and the
golden switch/start-bit/iterative corpus.  It does not import the package."""

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from variant_inputs import words  # noqa: E402
from test_oracle_variants import RUNS  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K(cuda):
    spec = importlib.util.spec_from_file_location("binarsort_cuda", os.path.join(HERE, "..", "integration", "_cuda.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert "paper_0811_3448_b200" not in m.__dict__
    return m


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_partition_worked_example(K):
    """tests/test_kernels.py:45-52: [B,4,0,0,7,A,C,E] at width 4, bit 0."""
    a = np.array([0xB, 0x4, 0x0, 0x0, 0x7, 0xA, 0xC, 0xE], dtype=np.uint32)
    c = K.new_counters()
    split = K.partition_words(a, 0, 7, 0, 4, c)
    assert split == 4 and a.tolist() == [0x7, 0x4, 0x0, 0x0, 0xA, 0xC, 0xE, 0xB]
    assert c.tolist()[:2] == [8, 4]


def test_range_sorted(K):
    """tests/test_kernels.py:78-82."""
    assert K.range_sorted_words(np.array([1, 2, 2, 3], dtype=np.uint32), 0, 3)
    assert not K.range_sorted_words(np.array([1, 3, 2], dtype=np.uint32), 0, 2)
    assert K.range_sorted_words(np.array([5], dtype=np.uint32), 0, 0)


def test_sortedness_check_stops_on_sorted_input(K):
    """tests/test_kernels.py:70-76: the scan makes a sorted input strictly cheaper."""
    base = np.arange(1000, dtype=np.uint32)
    slow, fast = K.new_counters(), K.new_counters()
    a = base.copy()
    K.sort_words(a, 0, 999, 0, 32, False, 0, 0, False, slow, 1)
    b = base.copy()
    K.sort_words(b, 0, 999, 0, 32, True, 4, 0, False, fast, 1)
    assert np.array_equal(a, base) and np.array_equal(b, base)
    assert fast[0] < slow[0]


def test_iterative_matches_recursive(K):
    """tests/test_kernels.py:55-68."""
    rng = np.random.default_rng(9)
    for n in (2, 17, 500, 3000):
        x = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
        a, b = x.copy(), x.copy()
        K.sort_words(a, 0, n - 1, 0, 32, False, 0, 0, False, K.new_counters(), 1)
        c = K.new_counters()
        K.sort_words_iterative(b, 0, n - 1, 32, c)
        assert np.array_equal(a, b) and c[3] <= 2 * (32 + 1)


def test_golden_corpus_through_the_binding(K):
    with open(os.path.join(HERE, "golden", "golden_variants.json")) as fh:
        gv = json.load(fh)
    for case in gv["kernel_variants"][::3]:  # a third of the corpus keeps this quick
        x = words(case["kind"], case["bits"], case["width"], case["n"], case["seed"])
        n, w = case["n"], case["width"]
        for name, (loop, chk, streak, checked, pos, depth) in RUNS.items():
            a = x.copy()
            c = K.new_counters()
            K.sort_words(a, 0, n - 1, pos, w, loop, chk, streak, checked, c, depth)
            want = case["runs"][name]
            assert sha(a) == want["output_sha"] and c.tolist() == want["counters"], (case["seed"], name)
        a = x.copy()
        c = K.new_counters()
        K.sort_words_iterative(a, 0, n - 1, w, c)
        want = case["runs"]["iterative"]
        assert sha(a) == want["output_sha"] and c.tolist() == want["counters"], case["seed"]
