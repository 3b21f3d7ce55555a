#!/bin/bash
# A/B on ONE box: previous vs current af_switch_mma.cuh
mkdir -p gpurun_out; : > gpurun_out/ab_switch.log
cp paper_2603_11873_b200/csrc/af_switch_mma.cuh /tmp/new.cuh
for v in new old new; do
  if [ $v = old ]; then cp scripts/old_af_switch_mma.cuh.txt paper_2603_11873_b200/csrc/af_switch_mma.cuh; else cp /tmp/new.cuh paper_2603_11873_b200/csrc/af_switch_mma.cuh; fi
  python -c "from paper_2603_11873_b200 import build; build.build(force=True)" > /dev/null 2>&1
  echo "version $v" >> gpurun_out/ab_switch.log
  timeout 200 python scripts/bench_switch.py --config 7b --modes mma --iters 8 2>&1 | grep mode >> gpurun_out/ab_switch.log
  timeout 200 python scripts/bench_switch.py --config 8b --modes mma --iters 8 2>&1 | grep mode >> gpurun_out/ab_switch.log
done
cp /tmp/new.cuh paper_2603_11873_b200/csrc/af_switch_mma.cuh
cat gpurun_out/ab_switch.log
