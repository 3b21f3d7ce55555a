#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_switch.py tests/test_gpu_chase.py tests/test_gpu_llama.py -q -x 2>&1 | tail -3
for k in 2 4; do
  echo "== 70b-tp8 k=$k"
  timeout 200 python scripts/bench_switch.py --config 70b-tp8 --layers 24 --k $k --modes mma --iters 4 2>&1 | grep '"mode"' | cut -c1-330
done
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 2>&1 | tail -1
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 --switch-mode from_pristine 2>&1 | tail -1
timeout 300 python bench.py --workload llama3-8b --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-3500
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-3500
