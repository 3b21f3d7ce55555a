#!/bin/bash
# K-chunked tcgen05 switch: correctness first, then timings (each step under its own timeout)
set -x
timeout 600 python -m pytest tests/test_gpu_switch.py -q -x -k "one_launch" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_switch.py tests/test_gpu_chase.py tests/test_gpu_llama.py -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_true_shapes.py -q -s --tb=line -k "llama3 or 70b or 13b" 2>&1 | grep -v "^$" | cut -c1-700 | tail -12
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 2>&1 | tail -2
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 --switch-mode from_pristine 2>&1 | tail -2
timeout 300 python bench.py --workload llama3-8b --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-2500
