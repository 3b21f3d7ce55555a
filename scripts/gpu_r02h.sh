#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_switch.py tests/test_gpu_chase.py -q -x 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_properties.py -q 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_true_shapes.py -q -s --tb=line -k "tp4 or tp8" 2>&1 | grep -v "^$" | cut -c1-500 | tail -8
for tp in 1 2 4 8; do timeout 300 python scripts/bench_shard.py llama2-7b --tp $tp --steps 20 2>&1 | tail -1; done
for tp in 2 4 8; do timeout 300 python scripts/bench_shard.py llama2-13b --tp $tp --steps 20 2>&1 | tail -1; done
