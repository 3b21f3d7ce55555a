#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_chase.py tests/test_gpu_llama.py -q -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_true_shapes.py -q -s --tb=short -k "bench" 2>&1 | grep -v "^$" | cut -c1-500 | tail -8
AF_CALIBRATE=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
timeout 600 python scripts/timeline_chase.py --ctx 1024 --show 17 2>&1 | tail -40
