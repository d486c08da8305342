"""Summarise an ncu launch list (gpu__time_duration + dram bytes) to the last sort's launches.

    python tools/launch_summary.py gpurun_out/TAG/launches.csv > profiles/rNN_launches.csv

The list comes from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv python bench.py --steps 1 ...`;
the last sort starts at the last init_kernel launch.  Per-launch times are
cold-cache and serialised, so the SHARE column is what compares with bench.py.
"""
import csv
import io
import sys
from collections import OrderedDict


def main(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    launches = OrderedDict()
    for r in rows:
        d = launches.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = list(launches)
    starts = [i for i in ids if launches[i]["name"].split("(")[0].split("<")[0].split()[-1] == "init_kernel"]
    last = [i for i in ids if i >= starts[-1]] if starts else ids
    total = sum(launches[i].get("gpu__time_duration.sum", 0) for i in last)
    print("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none")
    print(f"# source: {path}; last sort ({len(last)} launches) of the timed step, total {total / 1e3:.1f} us")
    print("# cold-cache serialised per-launch times: compare SHARES, not absolutes")
    print("kernel,duration_us,share,dram_read_GB,dram_write_GB")
    for i in last:
        d = launches[i]
        name = d["name"].replace("void ", "").split("(")[0]
        t = d.get("gpu__time_duration.sum", 0)
        print(f"\"{name}\",{t / 1e3:.1f},{t / total:.3f},{d.get('dram__bytes_read.sum', 0) / 1e9:.3f},"
              f"{d.get('dram__bytes_write.sum', 0) / 1e9:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
