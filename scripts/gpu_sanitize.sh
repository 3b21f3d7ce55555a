#!/bin/bash
# compute-sanitizer (memcheck + racecheck + synccheck) over the tcgen05 paths at tiny shapes: chained switch + GEMV launches
# (phase barriers, deferred RMSNorm, weighted schedule), the K-chunked one-launch switch up to 256 stacked ranks, ragged
# partial tiles, the decode attention (cp.async staging), whole Llama-block decode steps (graph and eager), the three-piece
# split of the gated rows and the tensor-parallel push step (PEERS instantiation, one rank as its own peer: the two-rank test
# needs two launches resident together, which the sanitizer's serialised launches cannot provide).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 5 \
     python -m pytest tests/test_gpu_chase.py tests/test_gpu_switch.py tests/test_gpu_llama.py tests/test_gpu_tp_push.py -q -m gpu -x --timeout 1200 \
       -k "chain_equals or deferred or prologues or validation or weighted or one_launch or (bank_switch and auto and (15 or 16)) or (decode_steps_against_oracle and chase and inplace) or split_attention or three_piece or engine_with_push or push_step_replays" \
       > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Race|Invalid|hazard" gpurun_out/sanitize_$tool.log | head -8
done
