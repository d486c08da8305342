#!/bin/bash
# Turn one measurement round (gpurun_out/TAG, made by tools/round_measure.sh) into the tracked profiles/ summaries.
# Usage: bash tools/collect_profiles.sh TAG rNN
set -eu
TAG=$1; R=$2
O=gpurun_out/$TAG
cp $O/configs.json profiles/${R}_configs.json
cp $O/pytest_gpu.log profiles/${R}_pytest_gpu.log
tail -1 $O/bench.json > profiles/${R}_bench.json
python tools/launch_summary.py $O/launches.csv > profiles/${R}_launches.csv
for d in $O/prof_*_details.csv; do
  k=$(basename $d _details.csv); k=${k#prof_}
  name=$(echo $k | sed 's/__.*//')   # dense_kernel__4608 -> dense_kernel
  {
    python tools/ncu_summary.py $d
    echo
    if [ -f $O/prof_${k}_sass.csv.gz ]; then
      gunzip -c $O/prof_${k}_sass.csv.gz > /tmp/_sass.csv
      python tools/sass_profile.py /tmp/_sass.csv
    fi
  } > profiles/${R}_ncu_prof_${name}.txt
done
python - "$O" <<'PY'
import csv, io, json, os, sys
O = sys.argv[1]
path = "profiles/traffic.json"
t = json.load(open(path))
for key, f in (("scatter_ws_kernel", "prof_scatter_ws_kernel_raw.csv"), ("dense_kernel", "prof_dense_kernel__4608_raw.csv"),
               ("hist16_kernel", "prof_hist16_kernel_raw.csv"), ("spread_kernel", "prof_spread_kernel_raw.csv")):
    p = os.path.join(O, f)
    if not os.path.exists(p):
        continue
    txt = open(p).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    hdr, units, val = rows[0], rows[1], rows[2]
    def get(name):
        i = hdr.index(name)
        v = float(val[i].replace(",", ""))
        u = units[i].lower()
        mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
                "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}.get(u, 1)
        return v * mult
    t[key] = {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
              "duration_ms": get("gpu__time_duration.sum"), "kernel": val[hdr.index("Kernel Name")][:120],
              "source": f"ncu --set full --clock-control none --import-source on, one launch ({O}; tools/round_measure.sh)"}
json.dump(t, open(path, "w"), indent=1)
print({k: (round(v["dram_read_bytes"] / 1e9, 3), round(v["dram_write_bytes"] / 1e9, 3), round(v["duration_ms"], 4)) for k, v in t.items()})
PY
