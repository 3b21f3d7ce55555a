#!/bin/bash
timeout 300 python scripts/bench_attn.py --ctx 1024 --splits 4,8,16,17,32
timeout 300 python scripts/bench_attn.py --ctx 128 --splits 1,2,4
timeout 300 python scripts/bench_attn.py --ctx 4096 --splits 16,32
AF_ATTN2=0 timeout 300 python scripts/bench_attn.py --ctx 1024 --splits 8
timeout 900 python -m pytest tests/test_gpu_decode_kernels.py tests/test_gpu_llama.py tests/test_gpu_chase.py -q -x 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-3500
