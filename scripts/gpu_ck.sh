#!/bin/bash
mkdir -p gpurun_out
for r in 1 2 3; do for u in 1 0; do
AF_UMMA=$u timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('AF_UMMA=$u chase', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), round(d['roofline'].get('ms_per_token'),4), 'switch', round(d['switch_us_per_token']))"
done; done 2>&1 | tee gpurun_out/umma_ab2.txt
