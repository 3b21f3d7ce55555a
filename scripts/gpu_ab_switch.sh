#!/bin/bash
# Same-box A/B of library builds on the standalone switch: scripts/gpu_ab_switch.sh libA.so libB.so ...
mkdir -p gpurun_out
for round in 1 2 3; do
for lib in "$@"; do
  export AF_LIB_PATH=$PWD/$lib
  timeout 300 python scripts/bench_switch.py --config 7b --modes mma --iters 8 2>&1 | grep '"mode"' | sed "s|^|$lib: |"
done; done 2>&1 | tee gpurun_out/ab_switch.txt
