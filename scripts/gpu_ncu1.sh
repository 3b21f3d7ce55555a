#!/bin/bash
mkdir -p gpurun_out
AF_NCU=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:switch_umma -s 17 -c 1 -o gpurun_out/prof_chase -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chase.log 2>&1
tail -3 gpurun_out/ncu_chase.log | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:switch_umma -s 2 -c 1 -o gpurun_out/prof_switch_umma -f \
   python scripts/bench_switch.py --config 7b --modes mma --iters 2 --warmup 1 > gpurun_out/ncu_switch_umma.log 2>&1
tail -2 gpurun_out/ncu_switch_umma.log | cut -c1-300
