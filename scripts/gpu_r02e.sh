#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_switch.py -q -x 2>&1 | tail -3
for k in 1 2 4; do
  for dbg in 0 32; do
    echo "== 70b-tp8 k=$k AF_DBG=$dbg"
    AF_DBG=$dbg timeout 200 python scripts/bench_switch.py --config 70b-tp8 --layers 24 --k $k --modes mma --iters 4 2>&1 | grep '"mode"' | cut -c1-330
  done
done
for ch in 0 1; do
  echo "== 8b AF_UMMA_CHUNK64=$ch"
  AF_UMMA_CHUNK64=$ch timeout 200 python scripts/bench_switch.py --config 8b --modes mma --iters 4 2>&1 | grep '"mode"' | cut -c1-330
done
echo "== 7b"
timeout 200 python scripts/bench_switch.py --config 7b --modes mma --iters 4 2>&1 | grep '"mode"' | cut -c1-330
