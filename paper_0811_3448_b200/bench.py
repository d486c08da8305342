"""Size-sweep benchmark harness and randomized differential check (drop-in for
``binarsort.bench`` and the CLI's ``bench``/``verify``), on the CUDA backend.

Reference: ``/root/reference/pkg/src/binarsort/bench.py`` (the plan, the
record and fit types, ``run_plan``'s warm-up-then-time method, the OLS fit
and the ``size,mean_ns,min_ns,max_ns`` CSV; bench.py:32-174) and
``cli.py:125-157,188-225`` (``cmd_bench``, ``cmd_verify``).  Same names,
fields, validation messages and CSV bytes, so the reference's schema tests
hold unchanged.  Additions:

* ``BenchPlan.timing``: ``"host"`` (default, the reference's method: a host
  array in, ``perf_counter_ns`` around the whole public call -- copies
  included) or ``"device"`` (input resident on the GPU, CUDA events around
  the device sort only, nanoseconds).
* ``verify``'s expected order comes from an independent comparison sort
  (numpy on the codec's encoded words) standing in for the reference's
  ``reference_sort`` (``sorted`` with the codec's ``le``, oracle.py:160-189).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import core, variants
from .cases import MT19937, CaseSpec, generate_case
from .keys import KEY_KINDS, codec_for_kind

__all__ = ["VARIANTS", "BenchPlan", "BenchRecord", "FitResult", "run_plan", "fit_linear", "write_csv",
           "CSV_HEADER", "make_sorter", "verify"]

VARIANTS = ("recursive", "iterative", "optimized", "parallel")
TIMINGS = ("host", "device")

CSV_HEADER = "size,mean_ns,min_ns,max_ns"


@dataclass
class BenchPlan:
    """Sweep configuration: sizes, iterations per size, data seed, variant (bench.py:37-66)."""

    start_size: int
    end_size: int
    step: int
    granularity: int
    seed: int = 0
    key_kind: str = "unsigned32"
    variant: str = "recursive"
    workers: int = 4
    timing: str = "host"

    def validate(self) -> None:
        if self.start_size < 1:
            raise ValueError("start_size must be >= 1")
        if self.end_size < self.start_size:
            raise ValueError("end_size must be >= start_size")
        if self.step < 1:
            raise ValueError("step must be >= 1")
        if self.granularity < 1:
            raise ValueError("granularity must be >= 1")
        if self.key_kind not in KEY_KINDS:
            raise ValueError(f"unknown key kind {self.key_kind!r}")
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.variant == "parallel" and self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.timing not in TIMINGS:
            raise ValueError(f"unknown timing {self.timing!r}")

    def sizes(self) -> range:
        return range(self.start_size, self.end_size + 1, self.step)


@dataclass
class BenchRecord:
    """Timing summary for one size; ``error`` set when the size failed."""

    size: int
    mean_ns: int = 0
    min_ns: int = 0
    max_ns: int = 0
    error: str | None = None


@dataclass
class FitResult:
    """Ordinary least squares of mean time against size."""

    slope: float
    intercept: float
    r_squared: float


def make_sorter(variant: str, codec, workers: int = 4):
    """Callable running one in-place sort of the chosen variant (bench.py:88-98)."""
    if variant == "recursive":
        return lambda seq: core.sort(seq, codec)
    if variant == "iterative":
        return lambda seq: variants.sort_iterative(seq, codec)
    if variant == "optimized":
        return lambda seq: variants.sort_optimized(seq, codec)
    if variant == "parallel":
        return lambda seq: variants.sort_parallel(seq, codec, workers)
    raise ValueError(f"unknown variant {variant!r}")


def _copy(seq):
    if isinstance(seq, np.ndarray):
        return seq.copy()
    return list(seq)


def _time_device(sorter, base):
    """One timed sort of a device-resident copy of ``base`` (CUDA events, ns)."""
    import torch

    raw = {4: np.int32, 8: np.int64}[base.dtype.itemsize]
    pristine = torch.from_numpy(base.view(raw).copy()).cuda()
    work = pristine.clone()
    if base.dtype.kind == "f":
        work = work.view(torch.float64)
    elif base.dtype.kind == "i":
        work = work.view(torch.int32 if base.dtype.itemsize == 4 else torch.int64)

    def once():
        work.view(pristine.dtype).copy_(pristine)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sorter(work)
        e1.record()
        torch.cuda.synchronize()
        return int(round(e0.elapsed_time(e1) * 1e6))

    return once


def run_plan(plan: BenchPlan) -> list[BenchRecord]:
    """Run the sweep; one record per size in plan order (bench.py:107-137).

    Per size: one generated case, one untimed warm-up sort, then
    ``granularity`` timed sorts of fresh copies.  Out-of-memory at a size
    produces an error record for that size rather than aborting the sweep.
    """
    plan.validate()
    codec = codec_for_kind(plan.key_kind)
    sorter = make_sorter(plan.variant, codec, plan.workers)
    records = []
    for size in plan.sizes():
        try:
            base = generate_case(CaseSpec(size, plan.key_kind, plan.seed))
            if plan.timing == "device" and isinstance(base, np.ndarray):
                once = _time_device(sorter, base)
                once()  # warm-up, untimed
                times = [once() for _ in range(plan.granularity)]
            else:
                sorter(_copy(base))  # warm-up, untimed
                times = []
                for _ in range(plan.granularity):
                    work = _copy(base)
                    t0 = time.perf_counter_ns()
                    sorter(work)
                    t1 = time.perf_counter_ns()
                    times.append(t1 - t0)
        except MemoryError:
            records.append(BenchRecord(size, error="allocation failed"))
            continue
        except RuntimeError as exc:  # CUDA out of memory
            if "out of memory" not in str(exc):
                raise
            records.append(BenchRecord(size, error="allocation failed"))
            continue
        records.append(BenchRecord(size, mean_ns=int(round(sum(times) / len(times))), min_ns=min(times),
                                   max_ns=max(times)))
    return records


def fit_linear(records: list[BenchRecord]) -> FitResult:
    """Least-squares line through (size, mean_ns); needs 2 distinct sizes (bench.py:140-154)."""
    points = [(r.size, r.mean_ns) for r in records if r.error is None]
    if len({s for s, _ in points}) < 2:
        raise ValueError("fit requires at least 2 records with distinct sizes")
    x = np.array([s for s, _ in points], dtype=np.float64)
    y = np.array([m for _, m in points], dtype=np.float64)
    xm, ym = x.mean(), y.mean()
    slope = float(((x - xm) * (y - ym)).sum() / ((x - xm) ** 2).sum())
    intercept = float(ym - slope * xm)
    ss_res = float(((y - (slope * x + intercept)) ** 2).sum())
    ss_tot = float(((y - ym) ** 2).sum())
    r_squared = 1.0 if ss_tot == 0.0 else 1.0 - ss_res / ss_tot
    return FitResult(slope, intercept, max(0.0, min(1.0, r_squared)))


def write_csv(records: list[BenchRecord], destination) -> None:
    """Write records (ascending size) as CSV to a path or text stream (bench.py:157-174).

    Error records carry no timings and are skipped.  A failed write raises
    OSError naming the destination.
    """
    rows = [CSV_HEADER]
    for r in sorted((r for r in records if r.error is None), key=lambda r: r.size):
        rows.append(f"{r.size},{r.mean_ns},{r.min_ns},{r.max_ns}")
    text = "\n".join(rows) + "\n"
    if hasattr(destination, "write"):
        destination.write(text)
        return
    try:
        with open(destination, "w", encoding="ascii") as fh:
            fh.write(text)
    except OSError as exc:
        raise OSError(f"cannot write CSV to {destination}: {exc}") from exc


# ---------------------------------------------------------------------------
# randomized differential (cli.py:188-225)
# ---------------------------------------------------------------------------

def _canonical(seq, key_kind: str) -> list:
    """Equality-faithful stand-ins (oracle.canonicalize, oracle.py:205-215)."""
    if key_kind == "float64":
        return [int(v) for v in np.asarray(seq, dtype=np.float64).view(np.uint64)]
    return [int(v) for v in seq]


def _expected(original, key_kind: str):
    """The codec order by an independent comparison sort of the encoded words."""
    a = np.asarray(original)
    if key_kind == "float64":
        u = a.astype(np.float64).view(np.uint64)
        enc = np.where(u >> np.uint64(63) == 1, ~u, u | np.uint64(1 << 63))
        return a[np.argsort(enc, kind="stable")]
    return np.sort(a, kind="stable")


def verify(cases: int, seed: int, key_kind: str = "unsigned32", variant: str = "recursive",
           workers: int = 4) -> tuple[int, tuple[int, int] | None]:
    """``cases`` random generate_case inputs (sizes 0..2048 from MT19937(seed)),
    each sorted by the chosen variant on the GPU and checked for order,
    permutation and the reference's Metrics bounds.  Returns
    (passed, first failure's (case seed, size) or None)."""
    if cases < 1:
        raise ValueError("--cases must be >= 1")
    if variant == "parallel" and workers < 1:
        raise ValueError("--workers must be >= 1")
    if key_kind == "bytestring":
        raise ValueError("bytestring keys use the reference's generic engine (outside the B200 hot path)")
    codec = codec_for_kind(key_kind)
    sorter = make_sorter(variant, codec, workers)
    master = MT19937(seed)
    passed = 0
    first = None
    for _ in range(cases):
        size = master.next_u32() % 2049
        case_seed = master.next_u32()
        original = generate_case(CaseSpec(size, key_kind, case_seed))
        work = _copy(original)
        m = sorter(work)
        want = _canonical(_expected(original, key_kind), key_kind)
        got = _canonical(work, key_kind)
        width = codec.width_for(original)
        ok = (got == want and sorted(got) == sorted(_canonical(original, key_kind))
              and m.bit_extractions <= width * size and m.swaps <= m.bit_extractions
              and m.max_depth <= width + 1)
        if ok:
            passed += 1
        elif first is None:
            first = (case_seed, size)
    return passed, first
