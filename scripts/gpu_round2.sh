#!/bin/bash
# GPU pass: parity tests (each file under its own timeout), smoke, contract bench, ncu launch list + full capture.
mkdir -p gpurun_out
rm -f gpurun_out/tests.log
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
for f in tests/test_gpu_router.py tests/test_gpu_switch.py tests/test_gpu_model.py tests/test_gpu_llama.py tests/test_gpu_decode_kernels.py; do
  echo "=== $f" >> gpurun_out/tests.log
  timeout 900 python -m pytest $f -q -m gpu --timeout 600 --timeout-method=thread >> gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
done
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "exit $?" >> gpurun_out/bench.err
if [ "$1" != "noncu" ]; then
AF_NCU=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:switch_mma -s 2 -c 1 -o gpurun_out/prof_switch -f \
   python scripts/bench_switch.py --config 7b --modes mma --iters 2 --warmup 1 > gpurun_out/ncu_switch.log 2>&1
AF_NCU=1 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"gemv_fused|gemv_tma|attn_decode" -s 10 -c 6 -o gpurun_out/prof_gemv -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemv.log 2>&1
fi
grep -E "passed|failed|exit" gpurun_out/tests.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
ls -la gpurun_out
