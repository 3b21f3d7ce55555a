#!/bin/bash
mkdir -p gpurun_out
timeout 200 python scripts/timeline_chase.py --show 99 > gpurun_out/tl_chain.txt 2>&1
cat gpurun_out/tl_chain.txt
