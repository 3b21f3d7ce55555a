#!/bin/bash
mkdir -p gpurun_out
for w in llama2-7b llama3-8b; do for m in chase separate; do
  timeout 600 python scripts/bench_sweep.py $w --forward-mode $m > gpurun_out/sweep_${w}_${m}.log 2>&1; cat gpurun_out/sweep_${w}_${m}.log | tail -8
done; done
timeout 600 python scripts/bench_sweep.py llama2-7b --switch-mode from_pristine > gpurun_out/sweep_llama2-7b_chase_from_pristine.log 2>&1; tail -7 gpurun_out/sweep_llama2-7b_chase_from_pristine.log
timeout 900 python bench.py --no-cpu-baseline --steps 20 --workload llama2-13b > gpurun_out/bench_13b.json 2> gpurun_out/bench_13b.err; tail -2 gpurun_out/bench_13b.err; cat gpurun_out/bench_13b.json | cut -c1-900
