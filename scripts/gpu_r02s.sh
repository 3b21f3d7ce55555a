#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_llama.py -q -x -k persistent 2>&1 | tail -2
for flag in "" "--persistent-forward"; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $flag 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('[$flag] decode_only tok/s', round(d['decode_only_tok_s'],1), 'frac', round(d['decode_only']['frac'],4), 'step ms', round(d['ms_per_step'],4))"
done
