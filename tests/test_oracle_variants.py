"""Pin the C oracle's drive forms (and the observer restatement) against the
reference's own outputs for every switch, start bit and word width
(tests/golden/golden_variants.json, made by running the reference)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from variant_inputs import words  # noqa: E402

RUNS = {
    "base": (False, 0, 0, False, 0, 1),
    "loop": (True, 0, 0, False, 0, 1),
    "loop_chk4": (True, 4, 0, False, 0, 1),
    "rec_chk1": (False, 1, 0, False, 0, 1),
    "rec_chk3_s2_d3": (False, 3, 2, False, 0, 3),
    "loop_chk2_checked": (True, 2, 1, True, 0, 2),
    "pos5_d2": (False, 0, 0, False, 5, 2),
    "pos3_loop_chk1": (True, 1, 0, False, 3, 1),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gv():
    with open(os.path.join(HERE, "golden", "golden_variants.json")) as fh:
        return json.load(fh)


def test_kernel_variants_oracle(gv, oracle_lib):
    o = oracle_lib
    for case in gv["kernel_variants"]:
        x = words(case["kind"], case["bits"], case["width"], case["n"], case["seed"])
        assert sha(x) == case["input_sha"]
        n, w = case["n"], case["width"]
        for name, (loop, chk, streak, checked, pos, depth) in RUNS.items():
            a = x.copy()
            c = o.new_counters()
            o.sort_words(a, 0, n - 1, pos, w, loop, chk, streak, checked, c, depth)
            want = case["runs"][name]
            assert sha(a) == want["output_sha"] and [int(v) for v in c] == want["counters"], (case["seed"], name)
        a = x.copy()
        c = o.new_counters()
        o.sort_words_iterative(a, 0, n - 1, w, c)
        want = case["runs"]["iterative"]
        assert sha(a) == want["output_sha"] and [int(v) for v in c] == want["counters"], case["seed"]


def test_variant_forms_oracle(gv, oracle_lib):
    o = oracle_lib
    for case in gv["variant_forms"]:
        x = words(case["kind"], case["bits"], case["width"], case["n"], case["seed"])
        n, w = case["n"], case["width"]
        for workers in (1, 3, 4, 8):
            a = x.copy()
            m = o.sort_parallel(a, workers, w)
            want = case["runs"][f"parallel{workers}"]
            assert sha(a) == want["output_sha"] and [int(v) for v in m] == want["metrics"], (case["seed"], workers)
        a = x.copy()
        c = o.new_counters()
        o.sort_words(a, 0, n - 1, 0, w, True, 4, 0, False, c, 1)
        want = case["runs"]["optimized_default"]
        assert sha(a) == want["output_sha"] and [int(v) for v in c] == want["metrics"]


def test_observer_traces_oracle(gv, oracle_lib):
    from oracle.levels import sort_levels

    for tr in gv["observer_traces"]:
        x = words(tr["kind"], tr["bits"], tr["width"], tr["n"], tr["seed"])
        assert sha(x) == tr["input_sha"]
        a = x.copy()
        ev = []
        lo, up, pos = tr.get("range", [0, tr["n"] - 1, 0])
        c = sort_levels(a, lo, up, pos, tr["width"], lambda p, b: ev.append([p, [list(t) for t in b]]))
        assert sha(a) == tr["output_sha"]
        assert [int(v) for v in c] == tr["metrics"]
        assert sha(np.frombuffer(json.dumps(ev).encode(), dtype=np.uint8)) == tr["events_sha"]
