#!/bin/bash
for pen in 1 0 2 3 1; do
AF_UNIT_PENALTY_UMMA=$pen timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('penalty $pen: ms_per_step', round(d['ms_per_step'],4), 'roof ms', round(d['roofline']['ms_per_token'],4), 'frac', round(d['roofline']['frac'],4))"
done
