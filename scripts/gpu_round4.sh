#!/bin/bash
# GPU pass for the chase schedule: every -m gpu test file, smoke, contract bench in both schedules,
# ncu launch list of the e2e region, one full capture of a chained switch + GEMV launch, timeline probe.
mkdir -p gpurun_out
rm -f gpurun_out/tests.log
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for f in tests/test_gpu_*.py tests/test_harness.py tests/test_io.py; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout 600 python -m pytest $f -q -m gpu --timeout 300 --timeout-method=thread >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --forward-mode separate --no-cpu-baseline > gpurun_out/bench_separate.json 2> gpurun_out/bench_separate.err
timeout 300 python scripts/timeline_chase.py --show 0,1,17,32 > gpurun_out/chase_timeline.txt 2>&1
if [ "$1" != "noncu" ]; then
AF_NCU=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 300 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
AF_NCU=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:switch_u?mma -s 17 -c 1 -o gpurun_out/prof_chase -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chase.log 2>&1
fi
grep -E "passed|failed|exit" gpurun_out/tests.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/bench_separate.json
tail -3 gpurun_out/ncu_launches.log gpurun_out/ncu_chase.log
ls -la gpurun_out
