#!/bin/bash
# Fast GPU check while tuning a kernel: focused parity tests + bench phases.
# Usage: gpurun --timeout 900 -- 'bash tools/quick_gpu.sh [extra pytest -k expr]'
K=${1:-"distributions or random_sizes or edge or dense or hist16 or kv or sorted_input or sequence or signed or whole_input"}
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > /tmp/q_pytest.log 2>&1
grep -E "^(FAILED|E  )" /tmp/q_pytest.log | head -12; tail -1 /tmp/q_pytest.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > /tmp/q_bench.json 2> /tmp/q_bench.err || tail -3 /tmp/q_bench.err
python -c "
import json,sys
d=json.loads(open('/tmp/q_bench.json').read().strip().splitlines()[-1])
p=d['phases_ms']
print('ms/step %.4f  hist0 %.4f  scatter0 %.4f  scatter1 %.4f  local %.4f' % (d['ms_per_step'], p['hist0'], p['scatter0'], p['scatter1'], p['local']))" 2>/dev/null
