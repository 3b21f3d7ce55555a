#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/sweep_gemv.log
for defs in "-DAF_GEMV_MINB=4" "-DAF_GEMV_MINB=5" "-DAF_GEMV_MINB=6" "-DAF_GEMV_THREADS=128 -DAF_GEMV_MINB=8" "-DAF_GEMV_THREADS=128 -DAF_GEMV_MINB=10" "-DAF_GEMV_THREADS=512 -DAF_GEMV_MINB=2 -DAF_GEMV_RB=2"; do
  AF_NVCC_EXTRA="$defs" python -c "from paper_2603_11873_b200 import build; build.build(force=True, verbose=True)" 2>&1 | grep -A2 gemv_fused | grep -E "registers|spill" >> gpurun_out/sweep_gemv.log
  echo "variant [$defs]" >> gpurun_out/sweep_gemv.log
  timeout 200 python scripts/bench_decode.py llama2-7b 0 2>&1 | grep -E "variant|rror" >> gpurun_out/sweep_gemv.log
done
python -c "from paper_2603_11873_b200 import build; build.build(force=True)" > /dev/null 2>&1
cat gpurun_out/sweep_gemv.log
