#!/bin/bash
# Same-box A/B of library builds on the decode-only chain: scripts/gpu_ab_decode.sh libA.so libB.so ...
mkdir -p gpurun_out
for round in 1 2; do
for lib in "$@"; do
  export AF_LIB_PATH=$PWD/$lib
  timeout 120 python scripts/bench_decode.py llama2-7b 0 2>&1 | tail -2 | sed "s|^|$lib: |"
done; done 2>&1 | tee gpurun_out/ab_decode.txt
