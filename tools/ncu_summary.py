"""Summarise an `ncu --page details --csv` export (the metrics the roofline discussion uses)."""
import csv
import io
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "Mem Busy", "Max Bandwidth", "No Eligible"]


def summary(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    out = [f"# {rows[0]['Kernel Name']}"]
    seen = set()
    for r in rows:
        k = (r["Section Name"], r["Metric Name"])
        if r["Metric Name"] in WANT and k not in seen:
            seen.add(k)
            out.append(f"{r['Section Name'][:28]:28} | {r['Metric Name'][:40]:40} | {r['Metric Value']:>14} {r['Metric Unit']}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summary(p))
