#!/bin/bash
# sweep ring depth / store depth of the tensor-path switch kernel on the 7B table
mkdir -p gpurun_out; : > gpurun_out/sweep_switch.log
for st in 4 5 6 7 8 10; do for dp in 0 1 2 3; do
  echo "stages $st depth $dp" >> gpurun_out/sweep_switch.log
  AF_MMA_STAGES=$st AF_STORE_DEPTH=$dp timeout 120 python scripts/bench_switch.py --config 7b --modes mma --iters 8 --warmup 2 2>&1 | grep '"mode"' >> gpurun_out/sweep_switch.log
done; done
cat gpurun_out/sweep_switch.log
