#!/usr/bin/env python3
"""Generate tests/golden/golden_variants.json by running the REFERENCE itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_variants.py

Pins what only the exact reference-order engine can reproduce: the tie order
of UnsignedCodec(w) on wider words and of sub-range sorts from a start bit,
the counters of every drive form (kernels.sort_words with its switches,
sort_words_iterative, sort_optimized, sort_iterative, sort_parallel), the
level observer's traces (sort_with_observer / binar_sort_range), the unstable
order the generic engine gives tagged (key, payload) records, and the
signed/float codec orders on generate_case inputs.  Inputs come from
tests/golden/variant_inputs.py (numpy default_rng streams) and the
reference's own generate_case; each is pinned by its sha256.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from variant_inputs import KINDS, words  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    import binarsort
    from binarsort import (CaseSpec, Float64Codec, Metrics, OptimizationConfig, SignedCodec, SortRange,
                           UnsignedCodec, binar_sort_range, generate_case, kernels, sort, sort_iterative,
                           sort_optimized, sort_parallel, sort_with_observer)
    from binarsort.keys import KeyCodec

    assert binarsort.BACKEND == "numba", binarsort.BACKEND

    def mv(m):
        return [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]

    out = {"generator": "tests/golden/make_golden_variants.py", "reference_backend": binarsort.BACKEND}

    # --- kernel module: every switch, start bits, iterative --------------
    kcases = []
    seed = 100
    for bits, width in ((32, 32), (64, 64), (32, 12), (64, 40), (64, 32)):
        for n in (2, 3, 17, 300, 2000):
            for kind in KINDS:
                seed += 1
                x = words(kind, bits, width, n, seed)
                runs = {}
                for name, (loop, chk, streak, checked, pos, depth) in {
                    "base": (False, 0, 0, False, 0, 1),
                    "loop": (True, 0, 0, False, 0, 1),
                    "loop_chk4": (True, 4, 0, False, 0, 1),
                    "rec_chk1": (False, 1, 0, False, 0, 1),
                    "rec_chk3_s2_d3": (False, 3, 2, False, 0, 3),
                    "loop_chk2_checked": (True, 2, 1, True, 0, 2),
                    "pos5_d2": (False, 0, 0, False, 5, 2),
                    "pos3_loop_chk1": (True, 1, 0, False, 3, 1),
                }.items():
                    a = x.copy()
                    c = kernels.new_counters()
                    kernels.sort_words(a, 0, n - 1, pos, width, loop, chk, streak, checked, c, depth)
                    runs[name] = {"output_sha": sha(a), "counters": [int(v) for v in c]}
                a = x.copy()
                c = kernels.new_counters()
                kernels.sort_words_iterative(a, 0, n - 1, width, c)
                runs["iterative"] = {"output_sha": sha(a), "counters": [int(v) for v in c]}
                kcases.append({"bits": bits, "width": width, "n": n, "kind": kind, "seed": seed,
                               "input_sha": sha(x), "runs": runs})
    out["kernel_variants"] = kcases

    # --- public drive forms on numpy words (words_view path) ------------
    vcases = []
    seed = 500
    for bits, width in ((32, 32), (64, 64), (64, 32), (32, 20)):
        for n in (2, 5, 64, 1000, 5000):
            for kind in KINDS:
                seed += 1
                x = words(kind, bits, width, n, seed)
                runs = {}
                codec = UnsignedCodec(width)
                for name, fn in {
                    "sort": lambda a: sort(a, codec),
                    "iterative": lambda a: sort_iterative(a, codec),
                    "optimized_default": lambda a: sort_optimized(a, codec),
                    "optimized_loop_only": lambda a: sort_optimized(a, codec, OptimizationConfig(True, 0)),
                    "optimized_chk1": lambda a: sort_optimized(a, codec, OptimizationConfig(False, 1)),
                    "optimized_chk3": lambda a: sort_optimized(a, codec, OptimizationConfig(False, 3)),
                    "parallel1": lambda a: sort_parallel(a, codec, 1),
                    "parallel3": lambda a: sort_parallel(a, codec, 3),
                    "parallel4": lambda a: sort_parallel(a, codec, 4),
                    "parallel8": lambda a: sort_parallel(a, codec, 8),
                }.items():
                    a = x.copy()
                    m = fn(a)
                    runs[name] = {"output_sha": sha(a), "metrics": mv(m)}
                vcases.append({"bits": bits, "width": width, "n": n, "kind": kind, "seed": seed,
                               "input_sha": sha(x), "runs": runs})
    out["variant_forms"] = vcases

    # --- reference tests' hand cases through lists -----------------------
    lists = {}
    base = list(range(256))
    lists["range256_w32_optimized_chk1"] = mv(sort_optimized(list(base), UnsignedCodec(32),
                                                             OptimizationConfig(sortedness_check_after=1)))
    lists["range256_w32_sort"] = mv(sort(list(base), UnsignedCodec(32)))
    lists["range256_w8_optimized_noloop_chk1"] = mv(sort_optimized(
        list(base), UnsignedCodec(8), OptimizationConfig(passthrough_loop=False, sortedness_check_after=1)))
    lists["range256_w8_sort"] = mv(sort(list(base), UnsignedCodec(8)))
    nyb = [0xB, 0x4, 0x0, 0x0, 0x7, 0xA, 0xC, 0xE]
    for name, fn in {"iterative": sort_iterative, "optimized": sort_optimized}.items():
        s = list(nyb)
        lists[f"nybble_{name}"] = {"output": s, "metrics": mv(fn(s, UnsignedCodec(4)))}
        lists[f"nybble_{name}"]["output"] = s
    s = list(nyb)
    m = sort_parallel(s, UnsignedCodec(4), 4)
    lists["nybble_parallel4"] = {"output": s, "metrics": mv(m)}
    out["list_cases"] = lists

    # --- level observer traces -------------------------------------------
    traces = []
    seed = 900
    for bits, width, n, kind in ((32, 8, 8, "random"), (32, 4, 16, "ties"), (32, 32, 40, "random"),
                                 (32, 32, 40, "nearly"), (64, 64, 33, "lowvar"), (64, 32, 300, "ties"),
                                 (32, 32, 2000, "random"), (32, 16, 3000, "lowvar"), (64, 40, 1500, "sorted")):
        seed += 1
        x = words(kind, bits, width, n, seed)
        a = x.copy()
        ev = []
        m = sort_with_observer(a, UnsignedCodec(width), lambda pos, b: ev.append([pos, [list(t) for t in b]]))
        rec = {"bits": bits, "width": width, "n": n, "kind": kind, "seed": seed, "input_sha": sha(x),
               "output_sha": sha(a), "metrics": mv(m), "events_sha": sha(np.frombuffer(
                   json.dumps(ev).encode(), dtype=np.uint8)), "nevents": len(ev)}
        if n <= 40:
            rec["events"] = ev
        traces.append(rec)
    # observer on a sub-range from a start bit (binar_sort_range)
    x = words("random", 32, 32, 500, 977)
    a = x.copy()
    ev = []
    m = Metrics()
    binar_sort_range(a, SortRange(37, 420, 6), UnsignedCodec(32), m,
                     observer=lambda pos, b: ev.append([pos, [list(t) for t in b]]))
    traces.append({"bits": 32, "width": 32, "n": 500, "kind": "random", "seed": 977, "range": [37, 420, 6],
                   "input_sha": sha(x), "output_sha": sha(a), "metrics": mv(m),
                   "events_sha": sha(np.frombuffer(json.dumps(ev).encode(), dtype=np.uint8)), "nevents": len(ev)})
    # plain sub-range sorts from a start bit (numba-free generic recursion via lists is
    # identical; the word path is kernels.sort_words with pos > 0)
    sub = []
    for i, (lo, up, pos) in enumerate(((0, 499, 7), (13, 300, 2), (100, 101, 30), (5, 450, 16))):
        x = words("random", 32, 32, 500, 990 + i)
        a = x.copy()
        m = Metrics()
        binar_sort_range(a, SortRange(lo, up, pos), UnsignedCodec(32), m)
        sub.append({"seed": 990 + i, "range": [lo, up, pos], "input_sha": sha(x), "output_sha": sha(a),
                    "metrics": mv(m)})
    out["observer_traces"] = traces
    out["subrange_sorts"] = sub

    # --- tagged records: the generic engine's unstable order --------------
    class Tagged(KeyCodec):
        def __init__(self, w):
            self.width = w
            self._c = UnsignedCodec(w)

        def bit_at(self, rec, pos):
            return self._c.bit_at(rec[0], pos)

        def le(self, a, b):
            return a[0] <= b[0]

    tagged = []
    for i, (width, n, kind) in enumerate(((16, 500, "ties"), (32, 800, "random"), (8, 1200, "lowvar"),
                                          (32, 300, "sorted"))):
        x = words(kind, 32, width, n, 1200 + i)
        recs = [(int(k), j) for j, k in enumerate(x)]
        m = sort(recs, Tagged(width))
        tagged.append({"width": width, "n": n, "kind": kind, "seed": 1200 + i, "input_sha": sha(x),
                       "tags": [t for _, t in recs], "metrics": mv(m)})
    out["tagged_unstable"] = tagged

    # --- signed / float codecs on generate_case (tests/test_keys.py:163-188) --
    codecs = []
    for kind, n, seed in (("signed32", 5000, 3), ("signed32", 97, 11), ("float64", 5000, 4), ("float64", 97, 12)):
        x = np.asarray(generate_case(CaseSpec(n, kind, seed)))
        a = x.copy()
        m = sort(a, SignedCodec(32) if kind == "signed32" else Float64Codec())
        codecs.append({"kind": kind, "n": n, "seed": seed, "input_sha": sha(x), "output_sha": sha(a),
                       "metrics": mv(m)})
    specials = np.array([0.0, -0.0, 1.5, -3.25, np.inf, -np.inf, np.nan, -np.nan, 5e-324, -5e-324,
                         1.0, -1.0, 2.0, -2.0, 0.0, np.nan], dtype=np.float64)
    specials.view(np.uint64)[7] |= np.uint64(0x12345)  # a negative-sign NaN with a payload
    a = specials.copy()
    m = sort(a, Float64Codec())
    codecs.append({"kind": "float64_specials", "input_bits": [int(v) for v in specials.view(np.uint64)],
                   "output_bits": [int(v) for v in a.view(np.uint64)], "metrics": mv(m)})
    out["codec_cases"] = codecs

    path = os.path.join(HERE, "golden_variants.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes", file=sys.stderr)


if __name__ == "__main__":
    main()
