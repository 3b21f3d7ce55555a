#!/bin/bash
# Llama-3-8B (64 stacked ranks in a steady switch): tcgen05 kernel with the decoupled UP ring against mma.sync; 7B regression check.
mkdir -p gpurun_out
for f in tests/test_gpu_chase.py tests/test_gpu_switch.py tests/test_gpu_llama.py; do timeout 600 python -m pytest $f -x -q 2>&1 | tail -2; done
AF_UMMA_MAX_RANKS=64 timeout 600 python -m pytest tests/test_gpu_chase.py tests/test_gpu_switch.py tests/test_gpu_llama.py -x -q 2>&1 | tail -2
for round in 1 2; do
for mr in 32 64; do
  AF_UMMA_MAX_RANKS=$mr timeout 400 python bench.py --no-cpu-baseline --steps 20 --workload llama3-8b > gpurun_out/b8.json 2> gpurun_out/b8.err; tail -1 gpurun_out/b8.err
  python -c "
import json,sys;d=json.load(open('gpurun_out/b8.json'));print('8B max_ranks', sys.argv[1], 'chase', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'switch', round(d['switch_us_per_token'],1))" $mr
done; done 2>&1 | tee gpurun_out/ab_8b.txt
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b7.json 2> gpurun_out/b7.err; python -c "
import json;d=json.load(open('gpurun_out/b7.json'));print('7B chase', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'switch', round(d['switch_us_per_token'],1))" | tee -a gpurun_out/ab_8b.txt
