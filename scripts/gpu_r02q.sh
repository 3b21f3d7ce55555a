#!/bin/bash
for ch in 4 8; do
echo "== AF_UMMA_CH128=$ch"
AF_UMMA_CH128=$ch timeout 200 python scripts/bench_switch.py --config 70b-tp8 --layers 24 --k 2 --modes mma --iters 4 2>&1 | grep '"mode"' | cut -c1-250
AF_UMMA_CH128=$ch timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 --switch-mode from_pristine 2>&1 | tail -1 | cut -c1-250
done
AF_UMMA_CH128=8 timeout 600 python -m pytest tests/test_gpu_switch.py -q -x -k "one_launch" 2>&1 | tail -2
