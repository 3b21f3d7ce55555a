#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_decode_kernels.py tests/test_gpu_llama.py tests/test_gpu_chase.py -x -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'], 'decode-only tok/s', d['decode_only_tok_s'], d['decode_only_hbm_gbs'])"
timeout 300 python bench.py --no-cpu-baseline --steps 30 --forward-mode separate > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('separate', d['ms_per_step'], d['e2e']['ms_per_step'], 'switch', d['switch_us_per_token'], 'decode-only tok/s', d['decode_only_tok_s'], d['decode_only_hbm_gbs'])"
