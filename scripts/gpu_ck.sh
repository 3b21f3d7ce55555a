#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -6
for u in 1 0 1 0; do
AF_UMMA=$u timeout 400 python bench.py --no-cpu-baseline --steps 30 --workload llama3-8b > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('8B AF_UMMA=$u chase', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), round(d['roofline'].get('ms_per_token'),4), 'switch', round(d['switch_us_per_token']))"
done 2>&1 | tee gpurun_out/umma_8b_ab.txt
