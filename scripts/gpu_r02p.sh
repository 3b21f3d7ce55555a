#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_chase.py tests/test_gpu_switch.py tests/test_gpu_llama.py -q -x 2>&1 | tail -3
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('MLP epilogue: ms_per_step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'roof ms', round(d['roofline']['ms_per_token'],4), 'frac', round(d['roofline']['frac'],4), 'switch us', round(d['switch_us_per_token'],1))"
done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --workload llama3-8b 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('8b: ms_per_step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'switch us', round(d['switch_us_per_token'],1))"
timeout 300 python scripts/timeline_chase.py --ctx 1024 --show 17 2>&1 | grep -E "phase 1, first tile|launch 17|first entry"
