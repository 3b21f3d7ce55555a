#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --timeout 120 --timeout-method=thread 2>&1 | tail -6
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'], 'decode-only tok/s', d['decode_only_tok_s'])"
AF_UMMA=0 timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase mma.sync', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'])"
