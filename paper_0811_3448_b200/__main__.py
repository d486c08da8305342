"""``python -m paper_0811_3448_b200 {bench,verify,trace}`` -- the reference CLI's
benchmark, differential and trace subcommands on the CUDA backend.

Mirrors ``/root/reference/pkg/src/binarsort/cli.py`` (``cmd_bench``
cli.py:125-157, ``cmd_trace`` :160-185, ``cmd_verify`` :188-225): same
options, outputs and exit codes (0 success, 1 verification failure, 2 usage
error, 3 I/O error).  ``bench`` adds ``--timing {host,device}``.  The text
``sort`` subcommand (file parsing) is outside the hot path.
"""

from __future__ import annotations

import argparse
import sys

from .bench import BenchPlan, fit_linear, run_plan, verify, write_csv
from .core import sort_with_observer
from .keys import UnsignedCodec

TYPE_KINDS = {"u32": "unsigned32", "u64": "unsigned64", "i32": "signed32", "f64": "float64"}


def cmd_bench(args) -> int:
    plan = BenchPlan(start_size=args.start, end_size=args.end, step=args.step, granularity=args.granularity,
                     seed=args.seed, key_kind=TYPE_KINDS[args.type], variant=args.variant, workers=args.workers,
                     timing=args.timing)
    try:
        plan.validate()
    except ValueError as exc:
        print(f"error: invalid plan: {exc}", file=sys.stderr)
        return 2
    records = run_plan(plan)
    for rec in records:
        if rec.error is not None:
            print(f"size {rec.size}: {rec.error}", file=sys.stderr)
    try:
        write_csv(records, args.csv)
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    try:
        fit = fit_linear(records)
    except ValueError:
        print("fit: n/a (need at least 2 sizes)")
        return 0
    print(f"fit: slope={fit.slope:.6g} ns/element intercept={fit.intercept:.6g} ns r_squared={fit.r_squared:.6f}")
    return 0


def cmd_verify(args) -> int:
    try:
        passed, first = verify(args.cases, args.seed, TYPE_KINDS[args.type], args.variant, args.workers)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    print(f"{passed}/{args.cases} passed")
    if first is not None:
        print(f"first failure: seed={first[0]} size={first[1]}", file=sys.stderr)
        return 1
    return 0


def cmd_trace(args) -> int:
    limit = 1 << args.width
    values = []
    for token in args.values:
        try:
            v = int(token, 16)
        except ValueError:
            print(f"parse error: {token!r} is not a hex value", file=sys.stderr)
            return 2
        if not 0 <= v < limit:
            print(f"parse error: {token!r} does not fit in {args.width} bits", file=sys.stderr)
            return 2
        values.append(v)

    def fmt(indices) -> str:
        return " ".join(format(values[i], "X") for i in indices)

    def observer(pos, boundaries):
        print(f"bit {pos + 1}: " + "".join(f"[{fmt(range(lo, up + 1))}]" for lo, up in boundaries))

    print(f"begin: [{fmt(range(len(values)))}]")
    sort_with_observer(values, UnsignedCodec(args.width), observer)
    print(f"end: [{fmt(range(len(values)))}]")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_0811_3448_b200", description="B200 binar sort tools")
    sub = parser.add_subparsers(dest="subcommand", required=True)

    def add_common(p):
        p.add_argument("--type", choices=sorted(TYPE_KINDS), default="u32", help="element type (default u32)")
        p.add_argument("--variant", choices=("recursive", "iterative", "optimized", "parallel"),
                       default="recursive", help="sort variant (default recursive)")
        p.add_argument("--workers", type=int, default=4, help="workers for the parallel variant (default 4)")
        p.add_argument("--seed", type=int, default=0, help="data seed (default 0)")

    b = sub.add_parser("bench", help="size sweep, CSV size,mean_ns,min_ns,max_ns")
    b.add_argument("--start", type=int, required=True)
    b.add_argument("--end", type=int, required=True)
    b.add_argument("--step", type=int, required=True)
    b.add_argument("--granularity", type=int, default=5)
    b.add_argument("--csv", required=True, help="output CSV path ('-' for stdout is not supported)")
    b.add_argument("--timing", choices=("host", "device"), default="host",
                   help="host: the public call on a host array (reference method); device: CUDA events, "
                        "input resident")
    add_common(b)
    b.set_defaults(fn=cmd_bench)
    v = sub.add_parser("verify", help="randomized differential against an independent sort")
    v.add_argument("--cases", type=int, default=100)
    add_common(v)
    v.set_defaults(fn=cmd_verify)
    t = sub.add_parser("trace", help="per-bit-level trace of a small hex list")
    t.add_argument("--width", type=int, choices=(4, 8, 16, 32), required=True)
    t.add_argument("values", nargs="+")
    t.set_defaults(fn=cmd_trace)
    return parser


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:  # usage errors return 2 like the reference (cli.py exit codes)
        return int(exc.code) if isinstance(exc.code, int) else 2
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
