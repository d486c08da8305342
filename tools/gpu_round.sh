#!/bin/bash
# One GPU round-trip: parity tests, bench line, launch list, ncu captures of the top kernels.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_round.sh TAG [tests] [bench] [launches] [prof:KERNEL]...'
# prof:KERNEL profiles one launch of KERNEL (regex) in PROFCMD (default: a 1-step cfg2 bench run), skipping SKIP launches.
set -u
TAG=${1:-cur}; shift
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
for step in "$@"; do
  case $step in
    tests)
      timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
      tail -3 $O/pytest_gpu.log ;;
    bench)
      timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json ;;
    launches)
      timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
      echo "ncu launches rc=$?" ;;
    prof:*)
      K=${step#prof:}; KF=$(echo "$K" | tr -c "A-Za-z0-9_\n" "_")
      timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s ${SKIP:-0} -c 1 -o /tmp/prof_$KF \
        ${PROFCMD:-python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline} > $O/ncu_$KF.log 2>&1; echo "ncu $K rc=$?"
      ncu -i /tmp/prof_$KF.ncu-rep --page details --csv > $O/prof_${KF}_details.csv 2>&1
      ncu -i /tmp/prof_$KF.ncu-rep --page raw --csv > $O/prof_${KF}_raw.csv 2>&1
      ncu -i /tmp/prof_$KF.ncu-rep --page source --csv --print-source sass > $O/prof_${KF}_sass.csv 2>&1
      gzip -f $O/prof_${KF}_sass.csv; rm -f /tmp/prof_$KF.ncu-rep ;;
    *) eval "$step" ;;
  esac
done
