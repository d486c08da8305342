#!/bin/bash
# Fast GPU check while tuning a kernel: focused parity tests + bench phases.
# Usage: gpurun --timeout 900 -- 'bash tools/quick_gpu.sh [extra pytest -k expr]'
K=${1:-"distributions or random_sizes or edge or dense or hist16 or kv or sorted_input or sequence or signed"}
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" 2>&1 | tail -2
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
p=d['phases_ms']
print('ms/step %.4f  hist0 %.4f  scatter0 %.4f  scatter1 %.4f  local %.4f' % (d['ms_per_step'], p['hist0'], p['scatter0'], p['scatter1'], p['local']))"
