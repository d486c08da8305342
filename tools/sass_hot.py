"""Top SASS instructions of an `ncu --page source --csv --print-source sass` export (.csv or .csv.gz):
by stall samples and by executed instructions; prints windows around the hottest PCs."""
import csv
import gzip
import io
import sys


def load(path):
    op = gzip.open if path.endswith(".gz") else open
    txt = op(path, "rt").read()
    i = txt.find('"Address"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def main(path, top=40):
    rows = load(path)
    tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    tot_i = sum(int(r["Instructions Executed"] or 0) for r in rows)
    print(f"instructions executed (warp): {tot_i}  stall samples: {tot_s}")
    idx = sorted(range(len(rows)), key=lambda k: -int(rows[k]["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for k in sorted(idx):
        r = rows[k]
        print(f"{k:5d} {int(r['Warp Stall Sampling (All Samples)']):7d} {int(r['Instructions Executed']):10d} "
              f"{r.get('L1 Wavefronts Shared','')[:8]:>8} {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
