#!/bin/bash
# Same-box A/B of library builds: scripts/gpu_ab.sh libA.so libB.so ...   (env passes through, e.g. AF_UMMA=0)
mkdir -p gpurun_out
for round in 1 2; do
for lib in "$@"; do
  export AF_LIB_PATH=$PWD/$lib
  echo "=== $lib (round $round)"
  timeout 300 python scripts/bench_switch.py --config 7b --modes mma --iters 6 2>&1 | grep '"mode"'
  timeout 120 python scripts/bench_chase_kernel.py --layers 6 2>&1 | grep -E "gu|o  "
  timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json;d=json.load(open('gpurun_out/b.json'));print('chase', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline'].get('ms_per_token'), 'switch', d['switch_us_per_token'])"
done; done 2>&1 | tee gpurun_out/ab.txt
