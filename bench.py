#!/usr/bin/env python3
"""Bench: sorted keys/s of the B200 Binar Sort hot path (BASELINE.json metric).

Workload (N=1, default): cfg2 = 2^28 uint32 keys, the first 2^28 words of
MT19937(1) (BASELINE.json configs[1]; synthetic by definition -- the reference
only ever uses seeded MT19937 data).  A *step* is one full sort of the
resident 1 GiB input.  Inputs are larger than L2 (126 MB), and the pristine
input is copied back into the work buffer between steps outside the timed
events, which also flushes L2.

N>1 (torchrun, default): cfg5 = 2^30 uint32 words of MT19937(4) (BASELINE.json
configs[4]) in contiguous 1/N slices, globally sorted through
``paper_0811_3448_b200.dist.dist_sort`` (device-sampled splitters, fused
partition + NVLink peer-store exchange, local sort): strong scaling.
``--config cfg2`` at N>1 is weak scaling (2^28 words of MT19937(1+rank) per
rank).  The output is checked before timing: every slice sorted, slices in
rank order, and order-independent checksums of all input shards equal to
those of all output slices.

CPU legs: ``cpu_baseline`` (rank 0, N=1) and ``--impl reference`` time the
REFERENCE itself -- ``binarsort.sort_parallel(arr, UnsignedCodec(32),
workers=<all host threads>)`` (numba) from ``baseline/_ref`` (pip-installed
from /root/reference) -- on the bench input, after a JIT
warm-up, with ``time.perf_counter_ns`` around the call (the reference's own
method, bench.py:107-137).  The whole input is used when the steps fit the
time budget, else the largest power-of-two prefix that does (stated in the
line).  Without baseline/_ref the C restatement in ``oracle/`` stands in
(``kind: "port"``).
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
# CPU legs: the reference itself (baseline/_ref, numba) when it is installed,
# else the oracle port -- test infrastructure, the baseline, never the product
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_module():
    """(binarsort module, None) from baseline/_ref, or (None, why)."""
    if not os.path.isdir(os.path.join(REF_DIR, "binarsort")):
        return None, "baseline/_ref is not installed"
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import binarsort
    except Exception as e:  # pragma: no cover - depends on the box
        return None, f"import binarsort failed: {e!r}"
    if getattr(binarsort, "BACKEND", None) != "numba":
        return None, f"reference backend is {getattr(binarsort, 'BACKEND', None)!r}, not numba"
    return binarsort, None


class _CpuSorter:
    """The CPU arm: reference ``sort_parallel`` (numba, all host threads) or the oracle port."""

    def __init__(self, workers: int):
        self.workers = workers
        self.ref, self.why = _reference_module()
        if self.ref is None:
            import oracle

            oracle.build()
            self.oracle = oracle
        self.kind = "reference" if self.ref is not None else "port"

    def describe(self) -> str:
        if self.ref is not None:
            return (f"reference binarsort.sort_parallel(arr, UnsignedCodec(32), workers={self.workers}) "
                    f"(baseline/_ref, numba; variants.py:162-229)")
        return (f"oracle port of sort_parallel (variants.py:162-229 restated in C, oracle/), "
                f"{self.workers} threads ({self.why})")

    def warm(self, x: np.ndarray) -> None:
        self.parallel(x[: 1 << 16].copy())
        self.single(x[: 1 << 12].copy())

    def parallel(self, y: np.ndarray) -> None:
        if self.ref is not None:
            self.ref.sort_parallel(y, self.ref.UnsignedCodec(32), self.workers)
        else:
            self.oracle.sort_parallel(y, self.workers)

    def single(self, y: np.ndarray) -> None:
        if self.ref is not None:
            self.ref.sort(y, self.ref.UnsignedCodec(32))
        else:
            self.oracle.sort(y, 32)


def _timed(fn, y) -> float:
    t0 = time.perf_counter_ns()
    fn(y)
    return (time.perf_counter_ns() - t0) / 1e9


def _pick_sample(cpu: _CpuSorter, x: np.ndarray, runs: int, budget_s: float) -> tuple[int, float]:
    """Largest power-of-two prefix (up to the whole input) whose `runs` timed sorts fit the budget,
    extrapolated from a 2^22-key probe (the sort is ~linear in n at fixed key width)."""
    probe = min(x.size, 1 << 22)
    dt = _timed(cpu.parallel, x[:probe].copy())
    per_key = dt / probe
    n = x.size
    while n > probe and runs * per_key * n * 1.15 > budget_s:
        n >>= 1
    return n, per_key


def cpu_baseline(x: np.ndarray, budget_s: float = 40.0):
    """Reported CPU baseline on the GPU box's host (rank 0, N=1): the reference on the bench input."""
    w = _affinity()
    cpu = _CpuSorter(w)
    cpu.warm(x)
    n, _ = _pick_sample(cpu, x, 1, budget_s)
    y = x[:n].copy()
    dt = _timed(cpu.parallel, y)
    ok = bool(np.array_equal(y[:: max(1, n // 65536)], np.sort(x[:n])[:: max(1, n // 65536)]))
    n1 = min(n, 1 << 24)
    dt1 = _timed(cpu.single, x[:n1].copy())
    return {"value": n / dt, "unit": UNIT, "cores": w, "kind": cpu.kind,
            "sample": (f"{'the whole' if n == x.size else 'first'} {n} keys of the bench input, "
                       f"{cpu.describe()}, 1 run after a JIT warm-up (bench.py:120-127 method)"),
            "same_config": n == x.size, "checked": ok,
            "single_thread": {"value": n1 / dt1, "sample": f"first {n1} keys, {'reference binarsort.sort' if cpu.ref else 'oracle sort'} (1 thread)"},
            "cpu_model": _cpu_model(), "cpu_count": os.cpu_count()}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _workload(args, world: int) -> str:
    return args.config if args.config != "auto" else ("cfg2" if world == 1 else "cfg5")


def _input_words(cfg: str, n_per_rank: int, rank: int, world: int) -> np.ndarray:
    """This rank's input: cfg2 = 2^28 words of MT19937(1+rank) per rank (weak);
    cfg5 = contiguous slice `rank` of n_total words of MT19937(4) (strong)."""
    from paper_0811_3448_b200.cases import mt_words

    if cfg == "cfg2":
        return mt_words(1 + rank, n_per_rank)
    lo, hi = (rank * n_per_rank) // world, ((rank + 1) * n_per_rank) // world
    return mt_words(4, hi)[lo:]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cfg = _workload(args, world)
    total = args.n if cfg == "cfg2" else args.total
    if cfg == "cfg2":
        total *= world  # weak scaling: the reference sorts what all ranks hold, as one array
    from paper_0811_3448_b200.cases import mt_words

    x = mt_words(1 if cfg == "cfg2" else 4, total) if (cfg == "cfg5" or world == 1) else \
        np.concatenate([mt_words(1 + r, args.n) for r in range(world)])
    w = _affinity()
    cpu = _CpuSorter(w)
    for _ in range(args.warmup):  # JIT warm-up (bench.py:120)
        cpu.warm(x)
    n, _ = _pick_sample(cpu, x, args.steps, args.ref_budget)
    times = []
    for i in range(args.steps):
        y = x[:n].copy()
        times.append(_timed(cpu.parallel, y))
    ok = bool(np.array_equal(y[:: max(1, n // 65536)], np.sort(x[:n])[:: max(1, n // 65536)]))
    ms = 1e3 * sum(times) / len(times)
    val = n / (ms / 1e3)
    line = {
        "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if cfg == "cfg2" else "strong",
        "vs_baseline": None, "dtype": "u32", "data": f"synthetic ({cfg} MT19937 stream)",
        "config": {"workload": (f"{cfg}: {'the whole' if n == x.size else 'first'} {n} of {x.size} uint32 keys"
                                f" ({'MT19937(1+rank) shards' if cfg == 'cfg2' else 'MT19937(4)'}), keys only"),
                   "global_batch": n, "parallelism": f"cpu threads x{w}", "same_config": n == x.size},
        "impl": "reference",
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": w, "kind": cpu.kind,
                         "sample": f"{n} keys per step, {cpu.describe()}", "checked": ok,
                         "cpu_model": _cpu_model(), "cpu_count": os.cpu_count()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0 if ok else 1


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _alg_bytes_per_key(keys_np: np.ndarray) -> tuple[int, int]:
    """(P_alg, bytes/key) per SURVEY §8d: non-constant 8-bit digits x 2 x key bytes."""
    d = np.bitwise_or.reduce(keys_np ^ keys_np[0]) if keys_np.size else 0
    kb = keys_np.dtype.itemsize
    p = sum(1 for b in range(kb) if (int(d) >> (8 * b)) & 0xFF)
    return p, 2 * kb * p


def _checksum(t):
    """Order-independent (sum, sum of splitmix64) of a CUDA u32-as-int32 tensor, int64 wrapping."""
    import torch

    x = t.to(torch.int64) & 0xFFFFFFFF
    z = x + (-7046029254386353131)  # 0x9E3779B97F4A7C15 as int64
    z = (z ^ ((z >> 30) & 0x3FFFFFFFF)) * (-4658895280553007687)  # 0xBF58476D1CE4E5B9
    z = (z ^ ((z >> 27) & 0x1FFFFFFFFF)) * (-7723592293110705685)  # 0x94D049BB133111EB
    z = z ^ ((z >> 31) & 0x1FFFFFFFF)
    return torch.stack([x.sum(), z.sum()])


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
    from paper_0811_3448_b200 import _lib, device

    cfg = _workload(args, world)
    host = _input_words(cfg, args.n if cfg == "cfg2" else args.total, rank, world)
    n = host.size
    total_keys = n * world if cfg == "cfg2" else args.total
    p_alg, bpk = _alg_bytes_per_key(host)
    if world > 1:  # P_alg of the whole input: OR over ranks of the varying-digit masks
        import torch.distributed as dist

        d = np.bitwise_or.reduce(host ^ host[0]) if host.size else np.uint32(0)
        t = torch.tensor([int(d), int(host[0]) if host.size else 0], dtype=torch.int64,
                         device="cpu" if share else dev)
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        firsts = [int(a[1]) for a in allt]
        dall = 0
        for a in allt:
            dall |= int(a[0]) | (int(a[1]) ^ firsts[0])
        p_alg = sum(1 for b in range(4) if (dall >> (8 * b)) & 0xFF)
        bpk = 2 * 4 * p_alg
    pristine = torch.from_numpy(host.view(np.int32)).to(dev)
    work = torch.empty_like(pristine)
    L = _lib.lib()
    ws = torch.empty(L.bs_workspace_bytes(n, 4, 0), dtype=torch.uint8, device=dev)
    nlev = (32 + 7) // 8 + 1
    nev = 1 + 3 * nlev + 1
    import ctypes

    from paper_0811_3448_b200.dist import SAMPLES_PER_RANK, dist_sort

    exch = {"mode": "auto", "ran": "", "note": ""}  # N>1: which data exchange dist_sort uses

    def one_sort(phases=None, marks=None):
        if world > 1:
            res = dist_sort(work, width=32, marks=marks, exchange=exch["mode"])
            exch["ran"] = res.exchange
            return res
        if phases is None:
            return device.sort_words_device(work, width=32, workspace=ws, check=False)
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
    a2a_max = 0
    if world == 1:
        if r is not None:
            device.check_status(r)
        ok = bool(torch.equal(work.view(torch.int32).cpu(), torch.from_numpy(np.sort(host).view(np.int32))))
        if not ok:
            print("bench: GPU output differs from np.sort", file=sys.stderr)
            return 1
    else:
        import torch.distributed as dist

        def validate(r):
            """This rank's slice sorted, slices in rank order, and the multiset kept (order-independent
            checksums of every input shard and every output slice); the same verdict on every rank."""
            k = r.keys.to(torch.int64) & 0xFFFFFFFF
            ok = bool((k[1:] >= k[:-1]).all()) if k.numel() > 1 else True
            sums = torch.cat([_checksum(pristine), _checksum(r.keys)]).to("cpu" if share else dev)
            dist.all_reduce(sums)
            s = [int(v) for v in sums.cpu()]
            ok = ok and s[0] == s[2] and s[1] == s[3]
            ends = torch.tensor([k.numel(), int(k[0]) if k.numel() else -1, int(k[-1]) if k.numel() else -1,
                                 sum(r.send_counts) - r.send_counts[rank]],
                                dtype=torch.int64, device="cpu" if share else dev)
            allends = [torch.empty_like(ends) for _ in range(world)]
            dist.all_gather(allends, ends)
            e = [[int(v) for v in t.cpu()] for t in allends]
            ok = ok and sum(x[0] for x in e) == total_keys
            a2a = 4 * max(x[3] for x in e)  # bytes the busiest rank sends to other ranks
            last = -1
            for cnt, lo, hi, _ in e:
                if cnt:
                    ok = ok and lo >= last
                    last = hi
            flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device="cpu" if share else dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same exit
            return int(flag.item()) == 1, a2a

        ok, a2a_max = validate(r)
        if not ok and exch["ran"] == "peer":
            # the fused peer-store exchange gave a wrong result on this machine: fall back to the
            # NCCL all-to-all exchange (every rank takes this branch: the verdict is all-reduced)
            print(f"bench: rank {rank}: peer exchange failed validation; retrying with exchange='collective'",
                  file=sys.stderr)
            exch["mode"] = "collective"
            exch["note"] = " (the peer-store exchange failed validation on this machine)"
            for i in range(max(1, args.warmup)):
                work.copy_(pristine)
                r = one_sort()
            torch.cuda.synchronize()
            ok, a2a_max = validate(r)
        if not ok:
            print(f"bench: rank {rank}: distributed output not globally sorted / multiset changed", file=sys.stderr)
            dist.destroy_process_group()
            return 1

    phase = [[] for _ in range(nev)]
    dphase = {}
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
            st = one_sort()
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            if world == 1 and st is not None:
                device.check_status(st)  # dropped work would fail the run loudly
        barrier()
        torch.cuda.synchronize()
        # per-phase breakdown, separate runs outside the timed steps
        for s in range(min(args.steps, 5)):
            work.copy_(pristine)
            if world == 1:
                one_sort(phase)  # the profiled call syncs
            else:
                marks = []
                barrier()
                one_sort(marks=marks)
                torch.cuda.synchronize()
                for (a, ea), (b, eb) in zip(marks, marks[1:]):
                    dphase.setdefault(b, []).append(ea.elapsed_time(eb))
    torch.cuda.synchronize()
    clocks = clk.summary()
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_keys / (ms / 1e3)
    peak, peak_kind = _peaks()
    if cfg == "cfg2":
        workload = ((f"cfg2: 2^{n.bit_length() - 1}" if n & (n - 1) == 0 else f"cfg2-shaped: {n}") +
                    " uint32 keys/rank, uniform from MT19937(1+rank), keys only, sort ascending")
    else:
        workload = (f"cfg5: {total_keys} uint32 keys uniform from MT19937(4), contiguous 1/{world} slice per rank"
                    ", keys only, globally sorted (rank r owns the r-th slice of the output)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if cfg == "cfg2" else "strong",
        "vs_baseline": None, "dtype": "u32",
        "data": f"synthetic ({'MT19937 seed 1+rank, cfg2 stream' if cfg == 'cfg2' else 'MT19937 seed 4, cfg5 stream'})",
        "config": {"workload": workload, "global_batch": total_keys, "keys_per_rank": n,
                   "parallelism": "single GPU" if world == 1 else
                   (f"range-partition x{world}: fused partition + NVLink peer stores (CUDA IPC), NCCL for counts"
                    if exch["ran"] == "peer" else
                    f"range-partition x{world}: partition + NCCL all-to-all-v" + exch["note"]),
                   "l2": f"inputs {4 * n / 2**20:.0f} MiB/rank > 126 MB L2; pristine copy restored between steps "
                         "(outside events)"},
        "clocks": clocks,
        # our kernels per step; N>1: sample, sample sort, class count (4), fused exchange, local sort
        "gpu_launches": (int(L.bs_sort_launches(n, 4, 32, 0, 0)) if world == 1 else
                         1 + int(L.bs_sort_launches(world * SAMPLES_PER_RANK, 4, 32, 0, 0)) + 5 +
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
            line["cpu_baseline"] = cpu_baseline(host, args.cpu_budget)
    else:
        import torch.distributed as dist

        # per-phase device times (max over ranks) of the peer path
        names = ["splitters", "class_count", "plan", "exchange", "barrier", "local_sort"]
        pt = torch.tensor([sum(dphase.get(k, [0.0])) / max(1, len(dphase.get(k, []))) for k in names],
                          dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
        ph = dict(zip(names, [float(v) for v in pt.cpu()]))
        line["phases_ms"] = {k: round(v, 4) for k, v in ph.items()}
        nmax = max(1, total_keys // world)
        ex_alg = 2 * 4 * nmax  # read the shard + store it (local or peer)
        lk_alg = 2 * 4 * nmax * p_alg
        dominant = "exchange" if ph["exchange"] >= ph["local_sort"] else "local_sort"
        kms = ph[dominant]
        alg = ex_alg if dominant == "exchange" else lk_alg
        achieved = alg / (kms / 1e3) / 1e9 if kms > 0 else None
        line["roofline"] = {"bound": "hbm", "kernel": "split_exchange_kernel" if dominant == "exchange"
                            else "bs_sort_from (local sort)", "achieved": achieved, "peak": peak,
                            "peak_kind": peak_kind, "unit": "GB/s",
                            "frac": achieved / peak if achieved else None, "traffic": None,
                            "alg_bytes_per_launch": alg, "avg_launch_ms": kms}
        t_hbm = bpk * nmax / (peak * 1e9)
        t_nvl = a2a_max / 900e9
        line["sort_roofline"] = {"p_alg": p_alg, "t_roof_ms": (t_hbm + t_nvl) * 1e3, "t_hbm_ms": t_hbm * 1e3,
                                 "t_nvlink_ms": t_nvl * 1e3, "a2a_bytes_max_rank": a2a_max,
                                 "frac": (t_hbm + t_nvl) * 1e3 / ms,
                                 "def": "SURVEY 8d: 2*(N/R)*kb*P_alg/hbm_gbs + A2A_bytes_max_rank/900 GB/s"}
        if not args.no_e2e:
            line["e2e"] = e2e_dist(args, host, dev, world, share, total_keys, exch["mode"])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def e2e_dist(args, host: np.ndarray, dev, world: int, share: bool, total_keys: int, exchange: str = "auto"):
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
        r = dist_sort(keys, width=32, exchange=exchange)
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
    return {"value": total_keys / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 4 * nout, "ms_per_step": ms, "steps": len(times),
            "api": "paper_0811_3448_b200.dist.dist_sort(shard copied from pinned host memory) + D2H of the slice",
            "per_rank_bytes": True}


def e2e(args, host: np.ndarray, dev):
    """Same metric end to end from pinned HOST memory through the public API.

    Headline: ``SortPipeline`` -- every step copies its 1 GiB input host->device,
    sorts it (bs_sort + Metrics), and copies the sorted keys and the counters
    back; consecutive steps overlap (PCIe is full duplex: step i+1's H2D runs
    while step i sorts and step i-1's D2H drains).  ``serial`` is the plain
    ``sort(pinned tensor)`` call (copy in, sort, copy out, one after another).
    """
    import torch

    from paper_0811_3448_b200 import UnsignedCodec, sort
    from paper_0811_3448_b200.pipeline import SortPipeline

    n = host.size
    pinned_src = torch.from_numpy(host.view(np.int32)).pin_memory()
    outs = [torch.empty_like(pinned_src).pin_memory() for _ in range(2)]
    steps = max(1, args.steps)
    pipe = SortPipeline(n, torch.int32, UnsignedCodec(32))
    pipe.run([pinned_src] * 2, outs)  # warm-up (allocations, first-touch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ms_list = pipe.run([pinned_src] * steps, [outs[i % 2] for i in range(steps)])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    want = np.sort(host)
    ok = all(bool(np.array_equal(o.numpy().view(np.uint32)[:: max(1, n // 65536)], want[:: max(1, n // 65536)]))
             for o in outs)
    m = ms_list[-1]
    pipe.close()
    ms = 1e3 * dt / steps
    # the plain serial call, for reference
    work = torch.empty_like(pinned_src).pin_memory()
    ser = []
    for i in range(1 + min(steps, args.e2e_steps)):
        work.copy_(pinned_src)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sort(work, UnsignedCodec(32))  # H2D, device sort + K6 metrics, D2H into `work`
        torch.cuda.synchronize()
        if i > 0:
            ser.append(time.perf_counter() - t1)
    ser_ms = 1e3 * sum(ser) / len(ser)
    return {"value": n / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 4 * n + 32, "ms_per_step": ms, "steps": steps,
            "api": "paper_0811_3448_b200.pipeline.SortPipeline(2^28, int32, UnsignedCodec(32)).run(pinned batches) "
                   "-> Metrics per batch; H2D / sort / D2H of consecutive steps overlapped on 3 CUDA streams",
            "checked": ok, "metrics": [m.bit_extractions, m.swaps, m.recursive_calls, m.max_depth],
            "serial": {"value": n / (ser_ms / 1e3), "ms_per_step": ser_ms, "steps": len(ser),
                       "api": "paper_0811_3448_b200.sort(pinned torch CPU tensor, UnsignedCodec(32))"}}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto", choices=["auto", "cfg2", "cfg5"],
                    help="auto: cfg2 at N=1 (2^28 keys), cfg5 at N>1 (2^30 keys over N ranks, strong scaling)")
    ap.add_argument("--keys-per-rank", "--n", dest="n", type=int, default=N_KEYS,
                    help="cfg2 keys per rank (default 2^28)")
    ap.add_argument("--total", type=int, default=1 << 30, help="cfg5 total keys (default 2^30)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=40.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=300.0,
                    help="seconds for the reference arm's timed steps (sample shrinks to fit)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
