#!/bin/bash
# Full GPU verification pass: every -m gpu test file, smoke(), and the contract bench line.
mkdir -p gpurun_out
rm -f gpurun_out/tests.log
for f in tests/test_gpu_*.py; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout 900 python -m pytest $f -q -m gpu --timeout 600 --timeout-method=thread >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
grep -E "passed|failed|exit|Error" gpurun_out/tests.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_ref.json
