#!/bin/bash
# build kernel variants on the box and time the worst-case (s = 2kr) switch on the 7B table
mkdir -p gpurun_out; : > gpurun_out/sweep_variants.log
for defs in "-DAF_WPROD=1 -DAF_STORERS=1" "-DAF_WPROD=2 -DAF_STORERS=1" "-DAF_WPROD=2 -DAF_STORERS=2" "-DAF_WPROD=4 -DAF_STORERS=2" "-DAF_WPROD=4 -DAF_STORERS=4" "-DAF_WPROD=2 -DAF_STORERS=2 -DAF_MR=64"; do
  AF_NVCC_EXTRA="$defs" python -c "from paper_2603_11873_b200 import build; build.build(force=True)" > /dev/null 2>&1
  for dp in 0 1; do
    echo "variant [$defs] depth $dp" >> gpurun_out/sweep_variants.log
    AF_STORE_DEPTH=$dp timeout 120 python scripts/bench_switch.py --config 7b --modes mma --iters 8 --warmup 2 2>&1 | grep '"mode"' >> gpurun_out/sweep_variants.log
  done
done
python -c "from paper_2603_11873_b200 import build; build.build(force=True)" > /dev/null 2>&1
cat gpurun_out/sweep_variants.log
