#!/bin/bash
# First GPU pass: parity tests (each file under its own timeout), smoke, switch bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for f in tests/test_gpu_router.py tests/test_gpu_switch.py tests/test_gpu_model.py; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout 600 python -m pytest $f -q -m gpu -x --timeout 300 --timeout-method=thread >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 600 python scripts/bench_switch.py --config 7b --modes mma,fma,exact --iters 5 > gpurun_out/bench_switch_7b.log 2>&1; echo "exit $?" >> gpurun_out/bench_switch_7b.log
timeout 300 python scripts/bench_switch.py --config tiny --modes mma,fma,exact --iters 20 > gpurun_out/bench_switch_tiny.log 2>&1
tail -5 gpurun_out/tests.log; cat gpurun_out/smoke.log | tail -3; cat gpurun_out/bench_switch_7b.log
