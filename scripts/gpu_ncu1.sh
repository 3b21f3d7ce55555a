#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:switch_mma -s 4 -c 1 -o gpurun_out/prof_gu -f \
   python scripts/bench_chase_kernel.py --layers 2 --iters 3 > gpurun_out/ncu_gu.log 2>&1
tail -3 gpurun_out/ncu_gu.log
