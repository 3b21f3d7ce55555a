#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py tests/test_gpu_switch.py tests/test_gpu_model.py -x -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -3
timeout 120 python scripts/bench_chase_kernel.py 2>&1 | grep AF_DBG
timeout 300 python scripts/bench_switch.py --config 7b --modes mma --iters 6 2>&1 | grep -i "mode\|GB"
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'], 'decode-only tok/s', d['decode_only_tok_s'])"
timeout 200 python scripts/timeline_chase.py --show 17 > gpurun_out/tl_chain.txt 2>&1; grep -E "p[0-9]\.|phase|unit|setup|span|blocked|step" gpurun_out/tl_chain.txt
