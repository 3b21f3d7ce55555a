#!/bin/bash
for dbg in 0 256 0 256; do
AF_DBG=$dbg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('AF_DBG=$dbg: ms_per_step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'roof ms', round(d['roofline']['ms_per_token'],4), 'frac', round(d['roofline']['frac'],4), 'switch_us', round(d['switch_us_per_token'],1))"
done
AF_DBG=256 timeout 600 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -q -x 2>&1 | tail -3
