#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -x -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -4
for d in 0 4; do AF_DBG=$d timeout 120 python scripts/bench_chase_kernel.py 2>&1 | grep AF_DBG; done | tee gpurun_out/chase_kernel.txt
timeout 200 python scripts/timeline_chase.py --show 17 > gpurun_out/tl_chain.txt 2>&1; cat gpurun_out/tl_chain.txt
timeout 200 python bench.py --no-cpu-baseline > gpurun_out/bench_chase.json 2> gpurun_out/bench_chase.err; python -c "
import json;d=json.load(open('gpurun_out/bench_chase.json'));print('chain', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['ms_per_token'])"
timeout 200 python bench.py --no-cpu-baseline --no-chain > gpurun_out/bench_chase_nc.json 2> gpurun_out/bench_chase_nc.err; python -c "
import json;d=json.load(open('gpurun_out/bench_chase_nc.json'));print('nochain', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['ms_per_token'])"
