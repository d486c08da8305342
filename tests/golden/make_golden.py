#!/usr/bin/env python3
"""Generate tests/golden/golden.json by running the REFERENCE itself.

Run in the build container (the reference lives at /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Everything recorded here is produced by the reference package (`binarsort`,
numba backend) -- its kernels, its sort entry points and its MT19937 -- on
seeded inputs that the tests regenerate independently (numpy generators,
documented per entry).  `--big` adds the full-size BASELINE.json configs
(2^28 / 2^30 keys; several minutes with sort_parallel on 8 threads).

Known answers pinned by the reference's own tests are included verbatim with
their file:line: tests/test_core.py:33-71,89-110,160-164,
tests/test_kernels.py:45-52, tests/test_oracle.py:10-17.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--out", default=os.path.join(HERE, "golden.json"))
    args = ap.parse_args()

    import binarsort
    from binarsort import (CaseSpec, Metrics, SortRange, UnsignedCodec, generate_case,
                           kernels, partition, sort, sort_parallel)
    from binarsort.keys import KeyCodec

    assert binarsort.BACKEND == "numba", binarsort.BACKEND
    out = {"generator": "tests/golden/make_golden.py", "reference_backend": binarsort.BACKEND}

    # --- known answers (reference tests) ---------------------------------
    nyb = [0xB, 0x4, 0x0, 0x0, 0x7, 0xA, 0xC, 0xE]
    seq = list(nyb)
    m = sort(seq, UnsignedCodec(4))
    out["nybble_sort"] = {"input": nyb, "output": seq,
                          "metrics": [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]}
    parts = []
    for inp, pos in ((nyb, 0), ([0x7, 0x4, 0x0, 0x0], 1), ([0xA, 0xC, 0xE, 0xB], 1), ([0, 0, 0], 0), ([0x8, 0x9], 0)):
        s = list(inp)
        mm = Metrics()
        r = partition(s, SortRange(0, len(s) - 1, pos), UnsignedCodec(4), mm)
        parts.append({"input": list(inp), "pos": pos, "output": s, "split": r.split,
                      "pass_through": r.pass_through, "extractions": mm.bit_extractions, "swaps": mm.swaps})
    out["partitions_w4"] = parts

    class Tagged(KeyCodec):
        def __init__(self, w):
            self.width = w
            self._c = UnsignedCodec(w)

        def bit_at(self, x, pos):
            return self._c.bit_at(x[0], pos)

        def le(self, a, b):
            return a[0] <= b[0]

    tagged = [(0x9, "a"), (0x1, "b"), (0x8, "c"), (0x2, "d"), (0x3, "e")]
    t = list(tagged)
    r = partition(t, SortRange(0, 4, 0), Tagged(4), Metrics())
    out["tagged_partition"] = {"keys": [k for k, _ in tagged], "tags": [g for _, g in tagged],
                               "out_tags": [g for _, g in t], "split": r.split}
    s = [0, 1]
    m = sort(s, UnsignedCodec(8))
    out["zero_one_w8"] = [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]

    # --- MT19937 stream heads + generate_case layouts -------------------
    heads = {}
    for seed in (5489, 1, 0, 2, 3, 4):
        heads[str(seed)] = [int(v) for v in binarsort.MT19937(seed).draw(12)]
    out["mt19937_heads"] = heads
    cases = {}
    for kind in ("unsigned32", "unsigned64", "signed32", "float64"):
        c = generate_case(CaseSpec(9, kind, 7))
        cases[kind] = [int(v) for v in np.asarray(c).view({4: np.uint32, 8: np.uint64}[np.asarray(c).itemsize])]
    out["generate_case_seed7_n9"] = cases

    # --- kernel sorts with counters: sizes 0..1500 (tests/test_kernels.py:34-42)
    ks = []
    for width, dt in ((32, np.uint32), (64, np.uint64)):
        rng = np.random.default_rng(21)
        for size in (0, 1, 2, 3, 17, 256, 1500):
            v = rng.integers(0, 2 ** width, size, dtype=np.uint64).astype(dt)
            a = v.copy()
            c = kernels.new_counters()
            if a.size > 1:
                kernels.sort_words(a, 0, a.size - 1, 0, width, False, 0, 0, False, c, 1)
            ks.append({"width": width, "size": size, "rng": "default_rng(21) sequential draws",
                       "input_sha": sha(v), "output_sha": sha(a), "counters": [int(x) for x in c],
                       "output_head": [int(x) for x in a[:4]]})
    out["kernel_sorts"] = ks

    # --- random partitions (exact unstable permutation) -----------------
    ps = []
    rng = np.random.default_rng(5)
    for it in range(60):
        n = int(rng.integers(1, 3000))
        w = int(rng.choice([8, 16, 32]))
        pos = int(rng.integers(0, w))
        v = rng.integers(0, 2 ** w, n, dtype=np.uint64).astype(np.uint32)
        a = v.copy()
        c = kernels.new_counters()
        split = int(kernels.partition_words(a, 0, n - 1, pos, w, c))
        ps.append({"n": n, "width": w, "pos": pos, "input_sha": sha(v), "output_sha": sha(a),
                   "split": split, "counters": [int(x) for x in c]})
    out["kernel_partitions"] = {"rng": "default_rng(5): n=integers(1,3000), w=choice([8,16,32]), "
                                       "pos=integers(0,w), keys=integers(0,2**w,n,uint64)->uint32",
                                "cases": ps}

    # --- cfg1: 2^20 u32 seed 0 (the oracle-run config) ------------------
    x = generate_case(CaseSpec(1 << 20, "unsigned32", 0))
    a = x.copy()
    t0 = time.time()
    m = sort(a, UnsignedCodec(32))
    out["cfg1"] = {"n": 1 << 20, "input_sha": sha(x), "output_sha": sha(a),
                   "metrics": [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth],
                   "seconds": round(time.time() - t0, 3)}
    print("cfg1 done", out["cfg1"]["seconds"], file=sys.stderr)

    if args.big:
        sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
        from paper_0811_3448_b200 import cases as C  # generators only (no GPU needed)

        big = {}
        w = os.cpu_count() or 8

        def run(name, arr, width):
            a = arr.copy()
            t0 = time.time()
            mm = sort_parallel(a, UnsignedCodec(width), w)
            big[name] = {"n": int(arr.size), "input_sha": sha(arr), "output_sha": sha(a),
                         "sort_parallel_workers": w,
                         "metrics_sort_parallel": [mm.bit_extractions, mm.swaps, mm.recursive_calls, mm.max_depth],
                         "seconds": round(time.time() - t0, 1)}
            print(name, big[name]["seconds"], file=sys.stderr, flush=True)
            return a

        run("cfg2", C.config2(), 32)
        for dist in ("uniform", "zipf", "low16"):
            run(f"cfg3_{dist}", C.config3(dist), 64)
        k, p = C.config4()
        packed = (k.astype(np.uint64) << np.uint64(32)) | p.astype(np.uint64)
        srt = run("cfg4_packed", packed, 64)
        big["cfg4_packed"]["keys_sha"] = sha((srt >> np.uint64(32)).astype(np.uint32))
        big["cfg4_packed"]["payload_sha"] = sha((srt & np.uint64(0xFFFFFFFF)).astype(np.uint32))
        del srt, packed, k, p
        x5 = C.config5("uniform")
        s5 = run("cfg5", x5, 32)
        big["cfg5_sorted"] = {"n": int(s5.size), "input_sha": sha(s5), "output_sha": sha(s5),
                              "note": "already sorted input = cfg5 output; sort is the identity"}
        r5 = s5[::-1].copy()
        run("cfg5_reverse", r5, 32)
        out["big"] = big

    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", args.out, file=sys.stderr)


if __name__ == "__main__":
    main()
