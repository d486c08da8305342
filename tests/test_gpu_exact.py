"""GPU parity of the exact reference-order engine (bs_exact_sort) and of every
drive form routed to it, against the reference's own outputs and counters
(tests/golden/golden_variants.json, made by tests/golden/make_golden_variants.py
running the reference) and against the C oracle on larger random inputs.

Restates, through this package, the assertions of the reference's
tests/test_kernels.py:55-82, tests/test_variants.py:35-177 and
tests/test_core.py:160-227 that concern the word path.
"""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

import paper_0811_3448_b200 as bs
from paper_0811_3448_b200 import _lib, cases, device, kernels
from paper_0811_3448_b200.core import Metrics, SortRange
from paper_0811_3448_b200.keys import Float64Codec, SignedCodec, UnsignedCodec
from paper_0811_3448_b200.variants import OptimizationConfig

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from variant_inputs import words  # noqa: E402
from test_oracle_variants import RUNS  # noqa: E402

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mv(m):
    return [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]


@pytest.fixture(scope="module")
def gv():
    with open(os.path.join(HERE, "golden", "golden_variants.json")) as fh:
        return json.load(fh)


def test_kernel_module_every_switch(cuda, gv):
    """kernels.sort_words with every switch / start bit / width, and sort_words_iterative."""
    for case in gv["kernel_variants"]:
        x = words(case["kind"], case["bits"], case["width"], case["n"], case["seed"])
        n, w = case["n"], case["width"]
        for name, (loop, chk, streak, checked, pos, depth) in RUNS.items():
            a = x.copy()
            c = kernels.new_counters()
            kernels.sort_words(a, 0, n - 1, pos, w, loop, chk, streak, checked, c, depth)
            want = case["runs"][name]
            assert sha(a) == want["output_sha"], (case["seed"], case["kind"], w, n, name)
            assert [int(v) for v in c] == want["counters"], (case["seed"], case["kind"], w, n, name)
        a = x.copy()
        c = kernels.new_counters()
        kernels.sort_words_iterative(a, 0, n - 1, w, c)
        want = case["runs"]["iterative"]
        assert sha(a) == want["output_sha"] and [int(v) for v in c] == want["counters"], case["seed"]


def test_drive_forms(cuda, gv):
    """sort / sort_iterative / sort_optimized / sort_parallel: output AND counters."""
    for case in gv["variant_forms"]:
        x = words(case["kind"], case["bits"], case["width"], case["n"], case["seed"])
        codec = UnsignedCodec(case["width"])
        forms = {
            "sort": lambda a: bs.sort(a, codec),
            "iterative": lambda a: bs.sort_iterative(a, codec),
            "optimized_default": lambda a: bs.sort_optimized(a, codec),
            "optimized_loop_only": lambda a: bs.sort_optimized(a, codec, OptimizationConfig(True, 0)),
            "optimized_chk1": lambda a: bs.sort_optimized(a, codec, OptimizationConfig(False, 1)),
            "optimized_chk3": lambda a: bs.sort_optimized(a, codec, OptimizationConfig(False, 3)),
            "parallel1": lambda a: bs.sort_parallel(a, codec, 1),
            "parallel3": lambda a: bs.sort_parallel(a, codec, 3),
            "parallel4": lambda a: bs.sort_parallel(a, codec, 4),
            "parallel8": lambda a: bs.sort_parallel(a, codec, 8),
        }
        for name, fn in forms.items():
            a = x.copy()
            m = fn(a)
            want = case["runs"][name]
            assert sha(a) == want["output_sha"], (case["seed"], case["kind"], case["width"], case["n"], name)
            assert mv(m) == want["metrics"], (case["seed"], case["kind"], case["width"], case["n"], name)


def test_reference_list_cases(cuda, gv):
    """tests/test_variants.py:75-92 and the nybble example through every form."""
    g = gv["list_cases"]
    base = list(range(256))
    fast = bs.sort_optimized(list(base), UnsignedCodec(32), OptimizationConfig(sortedness_check_after=1))
    slow = bs.sort(list(base), UnsignedCodec(32))
    assert mv(fast) == g["range256_w32_optimized_chk1"] and mv(slow) == g["range256_w32_sort"]
    assert fast.bit_extractions < slow.bit_extractions  # test_sorted_input_costs_strictly_less
    d = bs.sort_optimized(list(base), UnsignedCodec(8), OptimizationConfig(False, 1))
    assert mv(d) == g["range256_w8_optimized_noloop_chk1"] == g["range256_w8_sort"]
    seq = list(range(256))
    bs.sort_optimized(seq, UnsignedCodec(32), OptimizationConfig(sortedness_check_after=1))
    assert seq == list(range(256))
    nyb = [0xB, 0x4, 0x0, 0x0, 0x7, 0xA, 0xC, 0xE]
    for name, fn in (("iterative", bs.sort_iterative), ("optimized", bs.sort_optimized)):
        s = list(nyb)
        m = fn(s, UnsignedCodec(4))
        assert s == g[f"nybble_{name}"]["output"] and mv(m) == g[f"nybble_{name}"]["metrics"], name
    s = list(nyb)
    m = bs.sort_parallel(s, UnsignedCodec(4), 4)
    assert s == g["nybble_parallel4"]["output"] and mv(m) == g["nybble_parallel4"]["metrics"]


def test_observer_traces(cuda, gv):
    """sort_with_observer / binar_sort_range(observer=...) (core.py:146-239)."""
    for tr in gv["observer_traces"]:
        x = words(tr["kind"], tr["bits"], tr["width"], tr["n"], tr["seed"])
        a = x.copy()
        ev = []
        obs = lambda pos, b: ev.append([pos, [list(t) for t in b]])  # noqa: E731
        if "range" in tr:
            lo, up, pos = tr["range"]
            m = Metrics()
            bs.binar_sort_range(a, SortRange(lo, up, pos), UnsignedCodec(tr["width"]), m, observer=obs)
        else:
            m = bs.sort_with_observer(a, UnsignedCodec(tr["width"]), obs)
        assert sha(a) == tr["output_sha"], tr["seed"]
        assert mv(m) == tr["metrics"], tr["seed"]
        if "events" in tr:
            assert ev == tr["events"], tr["seed"]
        assert sha(np.frombuffer(json.dumps(ev).encode(), dtype=np.uint8)) == tr["events_sha"], tr["seed"]
    # tests/test_core.py:200-202: a single element fires no events
    ev = []
    bs.sort_with_observer(np.array([7], np.uint32), UnsignedCodec(8), lambda p, b: ev.append(p))
    assert ev == []


def test_subrange_sorts_from_a_start_bit(cuda, gv):
    for sub in gv["subrange_sorts"]:
        x = words("random", 32, 32, 500, sub["seed"])
        a = x.copy()
        lo, up, pos = sub["range"]
        m = Metrics()
        bs.binar_sort_range(a, SortRange(lo, up, pos), UnsignedCodec(32), m)
        assert sha(a) == sub["output_sha"] and mv(m) == sub["metrics"], sub["range"]


def test_tagged_records_reference_unstable_order(cuda, gv):
    """exact=True with values: the generic engine's order of (key, tag) records
    (tests/test_core.py:65-71 generalised)."""
    for tc in gv["tagged_unstable"]:
        x = words(tc["kind"], 32, tc["width"], tc["n"], tc["seed"])
        assert sha(x) == tc["input_sha"]
        k = x.copy()
        tags = np.arange(tc["n"], dtype=np.uint32)
        m = bs.sort(k, UnsignedCodec(tc["width"]), values=tags, exact=True)
        assert tags.tolist() == tc["tags"], tc["seed"]
        assert mv(m) == tc["metrics"], tc["seed"]


def test_signed_and_float_codecs_vs_reference(cuda, gv):
    """generate_case signed32/float64 and the special values (tests/test_keys.py:163-188)."""
    for cc in gv["codec_cases"]:
        if cc["kind"] == "float64_specials":
            a = np.array(cc["input_bits"], dtype=np.uint64).view(np.float64).copy()
            m = bs.sort(a, Float64Codec())
            assert [int(v) for v in a.view(np.uint64)] == cc["output_bits"]
            assert mv(m) == cc["metrics"]
            continue
        x = np.asarray(cases.generate_case(cases.CaseSpec(cc["n"], cc["kind"], cc["seed"])))
        assert sha(x) == cc["input_sha"]
        for exact in (None, True):
            a = x.copy()
            m = bs.sort(a, SignedCodec(32) if cc["kind"] == "signed32" else Float64Codec(), exact=exact)
            assert sha(a) == cc["output_sha"], (cc["kind"], exact)
            assert mv(m) == cc["metrics"], (cc["kind"], exact)


@pytest.mark.parametrize("bits,width", [(32, 32), (64, 64), (64, 32), (32, 24)])
def test_large_random_vs_oracle(cuda, oracle_lib, bits, width):
    """2^20 words: exact engine (optimised, iterative, parallel) vs the C oracle."""
    o = oracle_lib
    x = words("random", bits, width, 1 << 20, 7000 + bits + width)
    n = x.size
    for loop, chk in ((True, 4), (False, 2), (False, 0)):
        a, b = x.copy(), x.copy()
        c = kernels.new_counters()
        kernels.sort_words(a, 0, n - 1, 0, width, loop, chk, 0, False, c, 1)
        co = o.new_counters()
        o.sort_words(b, 0, n - 1, 0, width, loop, chk, 0, False, co, 1)
        assert np.array_equal(a, b) and np.array_equal(c, co), (loop, chk)
    a, b = x.copy(), x.copy()
    c = kernels.new_counters()
    kernels.sort_words_iterative(a, 0, n - 1, width, c)
    co = o.new_counters()
    o.sort_words_iterative(b, 0, n - 1, width, co)
    assert np.array_equal(a, b) and np.array_equal(c, co)
    a, b = x.copy(), x.copy()
    m = bs.sort_parallel(a, UnsignedCodec(width), 8)
    mo = o.sort_parallel(b, 8, width)
    assert np.array_equal(a, b) and mv(m) == [int(v) for v in mo]


def test_exact_engine_equals_fast_path_at_scale(cuda):
    """2^24 full-width keys: the exact engine and the digit sort agree (output and
    baseline counters), and the device path is the one that ran."""
    t = cuda
    x = cases.mt_words(1, 1 << 24)
    k1 = t.from_numpy(x.view(np.int32)).cuda()
    k2 = k1.clone()
    c1 = t.zeros(4, dtype=t.int64, device="cuda")
    c2 = t.zeros(4, dtype=t.int64, device="cuda")
    device.sort_words_device(k1, width=32, counters=c1)
    device.exact_sort_device(k2, width=32, mode=_lib.EX_REC, counters=c2)
    assert t.equal(k1, k2)
    assert t.equal(c1, c2)
    assert np.array_equal(k2.cpu().numpy().view(np.uint32), np.sort(x))
