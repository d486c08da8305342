"""Stall-reason totals, shared-memory wavefronts and the hottest SASS of an
`ncu --page source --csv --print-source sass` export (.csv or .csv.gz)."""
import collections
import csv
import gzip
import io
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    txt = op(path, "rt").read()
    i = txt.find('"Address"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def num(v):
    try:
        return float(v)
    except (TypeError, ValueError):
        return 0.0


def main(path, top=30):
    rows = load(path)
    stalls = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
    tot = collections.Counter()
    for r in rows:
        for k in stalls:
            tot[k] += num(r[k])
    ti = sum(num(r["Instructions Executed"]) for r in rows)
    wf = sum(num(r["L1 Wavefronts Shared"]) for r in rows)
    wfi = sum(num(r["L1 Wavefronts Shared Ideal"]) for r in rows)
    print(f"warp instructions {ti:.0f}   smem wavefronts {wf:.0f} (ideal {wfi:.0f})")
    s = sum(tot.values())
    print("stalls:", ", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in tot.most_common(8)))
    ops = collections.Counter()
    opw = collections.Counter()
    for r in rows:
        op = r["Source"].strip().split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else op[0])
        o = o.split(".")[0]
        ops[o] += num(r["Instructions Executed"])
        opw[o] += num(r["L1 Wavefronts Shared"])
    print("by opcode (warp instr, smem wavefronts):")
    for o, v in ops.most_common(18):
        print(f"   {o:10} {v:12.0f} {opw[o]:12.0f}")
    idx = sorted(range(len(rows)), key=lambda k: -num(rows[k]["Warp Stall Sampling (All Samples)"]))[:top]
    print("hottest (idx, samples, executed, wavefronts, top stall):")
    for k in sorted(idx):
        r = rows[k]
        st = max(stalls, key=lambda x: num(r[x]))
        print(f"{k:5d} {num(r['Warp Stall Sampling (All Samples)']):7.0f} {num(r['Instructions Executed']):10.0f} "
              f"{num(r['L1 Wavefronts Shared']):9.0f} {st[6:]:12} {r['Source'].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
