#!/bin/bash
# Full measurement round on one B200: GPU tests, bench line, launch list, every config, ncu --set full of the top kernels.
TAG=${1:-r02m}
O=gpurun_out/$TAG
mkdir -p $O
bash tools/gpu_round.sh $TAG tests bench launches
timeout 1500 python tools/bench_configs.py --reps 5 --out $O/configs.json > $O/configs.log 2>&1; tail -11 $O/configs.log
bash tools/gpu_round.sh $TAG "prof:scatter_ws_kernel" "prof:dense_kernel.*4608" "prof:hist16_kernel"
PROFCMD="python tools/bench_configs.py --only cfg3_uniform --reps 1 --warmup 0" bash tools/gpu_round.sh $TAG "prof:spread_kernel"
