#!/bin/bash
# compute-sanitizer over the tiny-shape chase / chain tests (memcheck + racecheck + synccheck).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 5 \
     python -m pytest tests/test_gpu_chase.py -q -m gpu -x --timeout 600 -k "chain_equals or deferred or prologues or validation" > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?"; grep -E "ERROR SUMMARY|passed|failed|Race|Invalid|hazard" gpurun_out/sanitize_$tool.log | head -8
done
