#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -x -q -m gpu --timeout 120 2>&1 | tail -3
timeout 200 python scripts/timeline_chase.py --show 17 > gpurun_out/tl_chain.txt 2>&1
grep -vE "Warning|nanvar|ret = " gpurun_out/tl_chain.txt | head -60
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'])"
