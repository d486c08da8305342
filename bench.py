#!/usr/bin/env python3
"""Bench: sorted keys/s of the B200 Binar Sort hot path (BASELINE.json metric).

Workload (N=1): cfg2 = 2^28 uint32 keys, the first 2^28 words of MT19937(1)
(BASELINE.json configs[1]; synthetic by definition -- the reference only ever
uses seeded MT19937 data).  A *step* is one full sort of the resident 1 GiB
input.  Inputs are larger than L2 (126 MB), and the pristine input is copied
back into the work buffer between steps outside the timed events, which also
flushes L2.  N>1 (torchrun): weak scaling, rank r holds 2^28 words of
MT19937(1+r) and the ranks globally sort the union through
``paper_0811_3448_b200.dist`` (sample splitters + NCCL all-to-all-v).

``--impl reference`` times the reference algorithm's CPU implementation: the
C restatement of the reference numba kernels in ``oracle/`` (the reference is
a Python/numba package; the restatement is line-for-line, see
oracle/binarsort_oracle.c), run as the reference's ``sort_parallel`` with all
host threads on a bounded sample of the cfg2 stream.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec (uint32, 2^28 keys) at 1/2/4/8 B200; fraction of HBM roofline"
UNIT = "keys/s"
N_KEYS = 1 << 28
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu launch list summary
    (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as fh:
            t = json.load(fh)[kernel]
        return int(t["dram_read_bytes"] + t["dram_write_bytes"])
    except Exception:
        return None


def _peaks():
    try:
        with open(PEAKS_PATH) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _affinity() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = f"/tmp/bs_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9:
                    rows.append(f)
        try:
            os.unlink(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU legs (oracle = test infrastructure: the checker/baseline, never the product)
# ---------------------------------------------------------------------------

def cpu_baseline(sample_keys: int = 1 << 25):
    import oracle

    oracle.build()
    x = _cfg2_words(sample_keys)
    w = _affinity()
    y = x.copy()
    oracle.sort_parallel(y[:1 << 16].copy(), w)  # warm
    t0 = time.perf_counter_ns()
    oracle.sort_parallel(y, w)
    dt = (time.perf_counter_ns() - t0) / 1e9
    n1 = sample_keys >> 3
    z = x[:n1].copy()
    t1 = time.perf_counter_ns()
    oracle.sort(z, 32)
    dt1 = (time.perf_counter_ns() - t1) / 1e9
    return {"value": sample_keys / dt, "unit": UNIT, "cores": w, "kind": "port",
            "sample": f"first {sample_keys} keys of cfg2 (MT19937 seed 1), oracle sort_parallel "
                      f"(variants.py:162-229 restated in C) with {w} threads, 1 run",
            "single_thread": {"value": n1 / dt1, "sample": f"first {n1} keys, oracle sort (1 thread)"},
            "cpu_model": _cpu_model()}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cfg2_words(n: int) -> np.ndarray:
    from paper_0811_3448_b200.cases import mt_words

    return mt_words(1, n)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import oracle

    oracle.build()
    sample = args.ref_sample
    x = _cfg2_words(sample)
    w = _affinity()
    oracle.sort_parallel(x[:1 << 16].copy(), w)
    times = []
    for i in range(args.warmup + args.steps):
        y = x.copy()
        t0 = time.perf_counter_ns()
        oracle.sort_parallel(y, w)
        dt = (time.perf_counter_ns() - t0) / 1e9
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    val = sample / (ms / 1e3)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (MT19937 seed 1, cfg2 stream)",
        "config": {"workload": f"cfg2 stream sample: first {sample} uint32 keys of MT19937(1), keys only",
                   "global_batch": sample, "parallelism": f"cpu threads x{w}"},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": w, "kind": "port",
                         "sample": f"first {sample} keys of cfg2, oracle sort_parallel with {w} threads per step",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _alg_bytes_per_key(keys_np: np.ndarray) -> tuple[int, int]:
    """(P_alg, bytes/key) per SURVEY §8d: non-constant 8-bit digits x 2 x key bytes."""
    d = np.bitwise_or.reduce(keys_np ^ keys_np[0]) if keys_np.size else 0
    kb = keys_np.dtype.itemsize
    p = sum(1 for b in range(kb) if (int(d) >> (8 * b)) & 0xFF)
    return p, 2 * kb * p


def run_gpu(args):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: BS_BENCH_SHARE_GPU=1 puts every rank on cuda:0 (gloo for the
    # host collectives) to exercise the N>1 path on a one-GPU box; never a
    # measurement (kernels of different ranks time-share one GPU)
    share = os.environ.get("BS_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_0811_3448_b200 import UnsignedCodec, _lib, device, sort
    from paper_0811_3448_b200.cases import mt_words

    n = args.n
    host = mt_words(1 + rank, n)
    p_alg, bpk = _alg_bytes_per_key(host)
    pristine = torch.from_numpy(host.view(np.int32)).to(dev)
    work = torch.empty_like(pristine)
    L = _lib.lib()
    ws = torch.empty(L.bs_workspace_bytes(n, 4, 0), dtype=torch.uint8, device=dev)
    nlev = (32 + 7) // 8 + 1
    nev = 1 + 3 * nlev + 1
    import ctypes

    def one_sort(phases=None):
        if world > 1:
            from paper_0811_3448_b200.dist import dist_sort

            return dist_sort(work, width=32)
        if phases is None:
            device.sort_words_device(work, width=32, workspace=ws)
            return None
        buf = (ctypes.c_float * nev)()
        nrec = ctypes.c_int(0)
        rc = L.bs_sort_profiled(work.data_ptr(), None, n, 4, 0, 32, 0, 0, ws.data_ptr(), ws.numel(),
                                torch.cuda.current_stream().cuda_stream, None, 1, buf, nev, ctypes.byref(nrec))
        _lib.check(rc)
        for i in range(nrec.value):
            phases[i].append(buf[i])
        return nrec.value

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    # warm-up (also checks correctness once)
    for i in range(args.warmup):
        work.copy_(pristine)
        r = one_sort()
    torch.cuda.synchronize()
    if world == 1:
        ok = bool(torch.equal(work.view(torch.int32).cpu(), torch.from_numpy(np.sort(host).view(np.int32))))
        if not ok:
            print("bench: GPU output differs from np.sort", file=sys.stderr)
            return 1
    else:  # this rank's slice sorted, slices in rank order, nothing lost
        import torch.distributed as dist

        k = r.keys.to(torch.int64) & 0xFFFFFFFF
        ok = bool((k[1:] >= k[:-1]).all()) if k.numel() > 1 else True
        ends = torch.tensor([k.numel(), int(k[0]) if k.numel() else -1, int(k[-1]) if k.numel() else -1],
                            dtype=torch.int64, device="cpu" if share else dev)
        allends = [torch.empty_like(ends) for _ in range(world)]
        dist.all_gather(allends, ends)
        e = [[int(v) for v in t.cpu()] for t in allends]
        ok = ok and sum(x[0] for x in e) == n * world
        last = -1
        for cnt, lo, hi in e:
            if cnt:
                ok = ok and lo >= last
                last = hi
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device="cpu" if share else dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same exit
        if int(flag.item()) == 0:
            print(f"bench: rank {rank}: distributed output not globally sorted", file=sys.stderr)
            dist.destroy_process_group()
            return 1

    phase = [[] for _ in range(nev)]
    step_ms = []
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for s in range(args.steps):
            work.copy_(pristine)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record()
            one_sort()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        barrier()
        torch.cuda.synchronize()
        if world == 1:  # per-phase breakdown, separate runs (the profiled call syncs)
            for s in range(min(args.steps, 5)):
                work.copy_(pristine)
                one_sort(phase)
    torch.cuda.synchronize()
    clocks = clk.summary()
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_keys = n * world
    value = total_keys / (ms / 1e3)
    peak, peak_kind = _peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (MT19937 seed 1+rank, cfg2 stream)",
        "config": {"workload": (f"cfg2: 2^{n.bit_length() - 1}" if n & (n - 1) == 0 else f"cfg2-shaped: {n}") +
                               " uint32 keys/rank, uniform from MT19937(1+rank), keys only, sort ascending",
                   "global_batch": total_keys, "keys_per_rank": n,
                   "parallelism": "single GPU" if world == 1 else
                   f"range-partition x{world}: fused partition + NVLink peer stores (CUDA IPC), NCCL for counts",
                   "l2": "inputs 1 GiB > 126 MB L2; pristine copy restored between steps (outside events)"},
        "clocks": clocks,
        # our kernels per step; N>1: sample, sample sort, class count (4), fused exchange, local sort
        "gpu_launches": (int(L.bs_sort_launches(n, 4, 32, 0, 0)) if world == 1 else
                         1 + int(L.bs_sort_launches(world * 4096, 4, 32, 0, 0)) + 5 +
                         int(L.bs_sort_launches(n, 4, 32, 0, 0))) * args.steps,
    }
    if world == 1:
        # phases: [init, (hist, plan, scatter) x nlev, local]
        names = ["init"] + [f"{k}{lv}" for lv in range(nlev) for k in ("hist", "plan", "scatter")] + ["local"]
        avg = {names[i]: (sum(v) / len(v)) for i, v in enumerate(phase[:len(names)]) if v}
        kinds = {"hist": 0.0, "plan": 0.0, "scatter": 0.0, "local": 0.0, "init": 0.0}
        for k, v in avg.items():
            kinds[k.rstrip("0123456789")] += v
        dominant = max(("scatter", "local", "hist"), key=lambda k: kinds[k])
        kname = {"scatter": "scatter_ws_kernel", "local": "dense_kernel", "hist": "hist16_kernel"}[dominant]
        if dominant == "scatter":
            durs = [avg[f"scatter{lv}"] for lv in range(nlev) if avg.get(f"scatter{lv}", 0) > 0.05]
            alg = 2 * 4 * n
        elif dominant == "local":
            durs = [avg["local"]]
            alg = 2 * 4 * n
        else:
            durs = [avg[f"hist{lv}"] for lv in range(nlev) if avg.get(f"hist{lv}", 0) > 0.05]
            alg = 4 * n
        kms = sum(durs) / len(durs)
        achieved = alg / (kms / 1e3) / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                            "traffic": _traffic(kname), "traffic_unit": "bytes per launch (ncu dram read+write)",
                            "alg_bytes_per_launch": alg, "avg_launch_ms": kms, "launches_averaged": len(durs)}
        t_roof = bpk * n / (peak * 1e9)
        line["sort_roofline"] = {"p_alg": p_alg, "alg_bytes": bpk * n, "t_roof_ms": t_roof * 1e3,
                                 "frac": t_roof * 1e3 / ms,
                                 "def": "SURVEY 8d: 2*N*kb*P_alg / hbm_gbs vs whole-sort time"}
        line["phases_ms"] = {k: round(v, 4) for k, v in avg.items() if v > 0.002}
        if not args.no_e2e:
            line["e2e"] = e2e(args, host, dev)
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_sample)
    if world > 1 and not args.no_e2e:
        line["e2e"] = e2e_dist(args, host, dev, world, share)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def e2e_dist(args, host: np.ndarray, dev, world: int, share: bool):
    """N>1 end to end through the public multi-GPU API: every rank copies its
    shard from pinned host memory, runs dist_sort, and reads its slice of the
    global order back into pinned host memory; max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_0811_3448_b200.dist import dist_sort

    n = host.size
    pinned_src = torch.from_numpy(host.view(np.int32)).pin_memory()
    pinned_out = torch.empty(2 * n + 4096, dtype=torch.int32).pin_memory()  # a slice is ~n keys
    times, nout = [], 0
    steps = max(1, min(args.steps, args.e2e_steps))
    for i in range(1 + steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        keys = pinned_src.to(dev, non_blocking=True)
        r = dist_sort(keys, width=32)
        out = pinned_out[:r.keys.numel()] if r.keys.numel() <= pinned_out.numel() else \
            torch.empty(r.keys.numel(), dtype=r.keys.dtype).pin_memory()
        out.copy_(r.keys, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        nout = r.keys.numel()
        if i > 0:
            times.append(dt)
    ms = torch.tensor([1e3 * sum(times) / len(times)], dtype=torch.float64, device="cpu" if share else dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    return {"value": n * world / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 4 * nout, "ms_per_step": ms, "steps": len(times),
            "api": "paper_0811_3448_b200.dist.dist_sort(shard copied from pinned host memory) + D2H of the slice",
            "per_rank_bytes": True}


def e2e(args, host: np.ndarray, dev):
    """Same metric through the public API with pinned HOST buffers (H2D + sort + D2H)."""
    import torch

    from paper_0811_3448_b200 import UnsignedCodec, sort

    n = host.size
    pinned_src = torch.from_numpy(host.view(np.int32)).pin_memory()
    work = torch.empty_like(pinned_src).pin_memory()
    times = []
    steps = max(1, min(args.steps, args.e2e_steps))
    for i in range(1 + steps):
        work.copy_(pinned_src)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = sort(work, UnsignedCodec(32))  # H2D, device sort + K6 metrics, D2H into `work`
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:
            times.append(dt)
    ok = bool(np.array_equal(work.numpy().view(np.uint32)[:: max(1, n // 4096)],
                             np.sort(host)[:: max(1, n // 4096)]))
    ms = 1e3 * sum(times) / len(times)
    return {"value": n / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 4 * n + 32, "ms_per_step": ms, "steps": len(times),
            "api": "paper_0811_3448_b200.sort(pinned torch CPU tensor, UnsignedCodec(32)) -> Metrics",
            "checked": ok, "metrics": [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth]}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--keys-per-rank", "--n", dest="n", type=int, default=N_KEYS, help="keys per rank (default 2^28 = cfg2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 25)
    ap.add_argument("--ref-sample", type=int, default=1 << 24)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
