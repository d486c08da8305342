"""Time every BASELINE.json configuration on one B200 (CUDA events, inputs resident).

For each config: keys/s (or pairs/s), the SURVEY 8d algorithmic roofline
(P_alg non-constant 8-bit digits x 2 x record bytes, vs MEASURED_PEAKS hbm_gbs)
and the fraction reached, plus a correctness check against np.sort /
np.argsort(stable).  Prints one JSON object per config and a markdown table.

    python tools/bench_configs.py [--reps 5] [--only cfg2,cfg4] [--out profiles/rNN_configs.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def p_alg(keys: np.ndarray) -> int:
    d = np.bitwise_or.reduce(keys ^ keys[0])
    return sum(1 for b in range(keys.dtype.itemsize) if (int(d) >> (8 * b)) & 0xFF)


def hbm_peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6521.1


def run(name: str, reps: int, with_phases: bool = True, warmup: int = 3):
    import torch

    from paper_0811_3448_b200 import _lib, device
    from paper_0811_3448_b200.cases import CONFIGS

    t0 = time.time()
    data = CONFIGS[name]()
    gen_s = time.time() - t0
    keys, vals = (data if isinstance(data, tuple) else (data, None))
    n = keys.size
    kb = keys.dtype.itemsize
    vb = 0 if vals is None else vals.dtype.itemsize
    raw = {4: torch.int32, 8: torch.int64}
    kdev0 = torch.from_numpy(keys.view(np.int32 if kb == 4 else np.int64)).cuda()
    vdev0 = None if vals is None else torch.from_numpy(vals.view(np.int32)).cuda()
    kdev = torch.empty_like(kdev0)
    vdev = None if vdev0 is None else torch.empty_like(vdev0)
    L = _lib.lib()
    ws = torch.empty(L.bs_workspace_bytes(n, kb, vb), dtype=torch.uint8, device="cuda")
    times = []
    for r in range(reps + warmup):  # first `warmup` runs untimed
        kdev.copy_(kdev0)
        if vdev is not None:
            vdev.copy_(vdev0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = device.sort_words_device(kdev, vdev, width=kb * 8, workspace=ws, check=False)
        e1.record()
        torch.cuda.synchronize()
        if st is not None:
            device.check_status(st)
        if r >= warmup:
            times.append(e0.elapsed_time(e1))
    phases = {}
    if with_phases:  # one extra profiled run: per-phase CUDA-event times
        import ctypes

        nlev = kb + 1
        nev = 1 + 3 * nlev + 1
        buf = (ctypes.c_float * nev)()
        nrec = ctypes.c_int(0)
        kdev.copy_(kdev0)
        if vdev is not None:
            vdev.copy_(vdev0)
        rc = L.bs_sort_profiled(kdev.data_ptr(), None if vdev is None else vdev.data_ptr(), n, kb, vb, kb * 8, 0, 0,
                                ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream, None, 1, buf, nev,
                                ctypes.byref(nrec))
        _lib.check(rc)
        names = ["init"] + [f"{k}{lv}" for lv in range(nlev) for k in ("hist", "plan", "scatter")] + ["local"]
        phases = {names[i]: round(buf[i], 4) for i in range(min(nrec.value, len(names))) if buf[i] > 0.003}
    got = kdev.cpu().numpy().view(keys.dtype)
    if vals is None:
        ok = bool(np.array_equal(got, np.sort(keys)))
    else:
        order = np.argsort(keys, kind="stable")
        ok = bool(np.array_equal(got, keys[order]) and
                  np.array_equal(vdev.cpu().numpy().view(vals.dtype), vals[order]))
    pa = p_alg(keys)
    alg = 2 * n * (kb + vb) * pa
    peak = hbm_peak()
    ms = float(np.median(times))
    t_roof = alg / (peak * 1e9) * 1e3
    del kdev0, kdev, ws, vdev0, vdev
    torch.cuda.empty_cache()
    return {"config": name, "n": n, "key_bytes": kb, "val_bytes": vb, "p_alg": pa,
            "ms_median": round(ms, 4), "ms_min": round(min(times), 4), "ms_max": round(max(times), 4),
            "keys_per_s": n / (ms / 1e3), "alg_bytes": alg, "t_roof_ms": round(t_roof, 4),
            "roofline_frac": round(t_roof / ms, 4), "peak_gbs": peak, "correct": ok,
            "gen_s": round(gen_s, 1), "phases_ms": phases}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args(argv)
    names = ["cfg1", "cfg2", "cfg3_uniform", "cfg3_zipf", "cfg3_low16", "cfg4", "cfg5", "cfg5_sorted",
             "cfg5_reverse"]
    if a.only:
        names = [x for x in names if x in a.only.split(",")]
    from bench import Clocks

    res = []
    for nm in names:
        with Clocks(0) as clk:
            r = run(nm, a.reps, warmup=a.warmup)
        r["clocks"] = clk.summary()
        print(json.dumps(r), flush=True)
        res.append(r)
    print("\n| config | n | P_alg | median ms | Gkeys/s | roofline ms | frac | correct |")
    print("|---|---|---|---|---|---|---|---|")
    for r in res:
        print(f"| {r['config']} | {r['n']} | {r['p_alg']} | {r['ms_median']:.3f} | {r['keys_per_s'] / 1e9:.1f} | "
              f"{r['t_roof_ms']:.3f} | {r['roofline_frac']:.2f} | {r['correct']} |")
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    return 0 if all(r["correct"] for r in res) else 1


if __name__ == "__main__":
    sys.exit(main())
