#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/tests.log
for f in tests/test_gpu_router.py tests/test_gpu_switch.py tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_decode_kernels.py; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout 900 python -m pytest $f -q -m gpu --timeout 600 --timeout-method=thread >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "exit $?" >> gpurun_out/bench.err
timeout 600 python scripts/bench_sweep.py llama3-8b > gpurun_out/sweep_8b.log 2>&1
timeout 600 python scripts/bench_sweep.py llama2-7b > gpurun_out/sweep_7b.log 2>&1
timeout 600 python scripts/bench_sweep.py llama2-7b --switch-mode from_pristine > gpurun_out/sweep_7b_pristine.log 2>&1
timeout 300 python scripts/bench_switch.py --config 8b --modes mma,fma --iters 5 > gpurun_out/bench_switch_8b.log 2>&1
timeout 300 python scripts/bench_switch.py --config 13b --modes mma --iters 5 > gpurun_out/bench_switch_13b.log 2>&1
grep -E "passed|failed|exit" gpurun_out/tests.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
cat gpurun_out/sweep_8b.log gpurun_out/sweep_7b.log gpurun_out/sweep_7b_pristine.log gpurun_out/bench_switch_8b.log gpurun_out/bench_switch_13b.log
