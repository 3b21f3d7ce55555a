#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/tests.log
for f in tests/test_gpu_switch.py tests/test_gpu_llama.py tests/test_gpu_model.py; do
  timeout 900 python -m pytest $f -q -m gpu --timeout 600 --timeout-method=thread 2>&1 | tail -4 >> gpurun_out/tests.log
done
cat gpurun_out/tests.log
for i in 1 2; do
echo "swizzled UP"; timeout 300 python scripts/bench_switch.py --config 8b --modes mma --iters 6 2>&1 | grep mode
echo "bulk UP"; AF_UP_SWIZZLE=0 timeout 300 python scripts/bench_switch.py --config 8b --modes mma --iters 6 2>&1 | grep mode
done
timeout 300 python scripts/bench_switch.py --config 7b --modes mma --iters 6 2>&1 | grep mode
