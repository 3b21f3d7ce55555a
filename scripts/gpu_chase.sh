#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -x -q -m gpu --timeout 120 --timeout-method=thread > gpurun_out/chase_tests.log 2>&1
rc=$?
echo "exit $rc" >> gpurun_out/chase_tests.log
tail -5 gpurun_out/chase_tests.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout 200 python bench.py --no-cpu-baseline > gpurun_out/bench_chase.json 2> gpurun_out/bench_chase.err; echo "exit $?"; tail -5 gpurun_out/bench_chase.err; cat gpurun_out/bench_chase.json
