#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_llama.py -q -x -k "persistent" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_chase.py tests/test_gpu_decode_kernels.py -q 2>&1 | tail -6
for fw in 0 1; do
AF_FW_PERSISTENT=$fw timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('AF_FW_PERSISTENT=$fw: ms_per_step', round(d['ms_per_step'],4), 'decode_only tok/s', round(d['decode_only_tok_s'],1), 'frac', round(d['decode_only']['frac'],4))"
done
AF_FW_PERSISTENT=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --forward-mode separate 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('separate persistent: ms_per_step', round(d['ms_per_step'],4), 'switch us', round(d['switch_us_per_token'],1))"
AF_FW_PERSISTENT=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --forward-mode separate 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('separate chained   : ms_per_step', round(d['ms_per_step'],4), 'switch us', round(d['switch_us_per_token'],1))"
