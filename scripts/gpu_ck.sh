#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -x -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -3
timeout 120 python scripts/bench_chase_kernel.py --plain 2>&1 | grep AF_DBG
timeout 120 python scripts/bench_chase_kernel.py 2>&1 | grep AF_DBG
for w in llama2-7b llama3-8b; do
for m in chase separate; do
timeout 300 python bench.py --no-cpu-baseline --steps 30 --workload $w --forward-mode $m > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('$w $m', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'], 'decode-only tok/s', d['decode_only_tok_s'])"
done; done | tee gpurun_out/workloads.txt
