#!/bin/bash
# Same-box A/B of library builds on the headline step only: scripts/gpu_ab_chase.sh libA.so libB.so ...
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_chase.py -x -q 2>&1 | tail -2
for round in 1 2 3; do
for lib in "$@"; do
  export AF_LIB_PATH=$PWD/$lib
  timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json,sys;d=json.load(open('gpurun_out/b.json'));print(sys.argv[1], 'chase', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), round(d['roofline'].get('ms_per_token'),4))" $lib
done; done 2>&1 | tee gpurun_out/ab_chase.txt
