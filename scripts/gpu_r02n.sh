#!/bin/bash
O=gpurun_out
timeout 600 python scripts/bench_sweep.py llama3-8b > $O/sweep_llama3-8b_chase.txt 2>&1
timeout 600 python scripts/bench_sweep.py llama3-8b --forward-mode separate > $O/sweep_llama3-8b_separate.txt 2>&1
timeout 600 python scripts/bench_sweep.py llama2-7b > $O/sweep_llama2-7b_chase.txt 2>&1
tail -8 $O/sweep_llama3-8b_chase.txt | cut -c1-200
# the N > 1 bench path rehearsed on ONE GPU (both ranks on cuda:0, collectives through gloo): plumbing only, timings mean nothing
PORT=$((20000 + RANDOM % 20000))
AF_DIST_BACKEND=gloo AF_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $PORT \
   bench.py --gpus 2 --steps 3 --warmup 3 > $O/rehearsal_tp2.json 2> $O/rehearsal_tp2.err
echo "rehearsal rc $?"; tail -1 $O/rehearsal_tp2.json | cut -c1-900; tail -5 $O/rehearsal_tp2.err | cut -c1-300
PORT=$((20000 + RANDOM % 20000))
AF_DIST_BACKEND=gloo AF_SHARE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $PORT \
   bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/rehearsal_tp2_ref.json 2>> $O/rehearsal_tp2.err
echo "reference rehearsal rc $?"; tail -1 $O/rehearsal_tp2_ref.json | cut -c1-300
