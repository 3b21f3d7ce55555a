#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_llama.py -q -x -k "prefill or generate" 2>&1 | tail -4
timeout 600 python scripts/bench_prefill.py llama2-7b --lengths 16,128,512,2048 --stepwise-max 128 2>&1 | tail -6
