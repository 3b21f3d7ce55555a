#!/bin/bash
# Round-2 evidence pass (one B200): every -m gpu test file, smoke, the contract bench (both arms, other workloads, the
# separate schedule), shard-alone timings, the standalone switch at 32 .. 256 stacked ranks, the decode attention, the
# chase timeline, and -- unless "noncu" -- the ncu launch list of the timed region and one full capture of a chained launch.
mkdir -p gpurun_out
O=gpurun_out
rm -f $O/tests.log
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
for f in tests/test_gpu_*.py tests/test_harness.py tests/test_io.py; do
  echo "=== $f" >> $O/tests.log
  timeout 1500 python -m pytest $f -q -m gpu -s --timeout 1200 --timeout-method=thread 2>&1 | grep -vE "^$" | cut -c1-400 | tail -14 >> $O/tests.log
done
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference_arm.json 2>> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --forward-mode separate --no-cpu-baseline > $O/bench_separate.json 2>> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --switch-mode from_pristine --no-cpu-baseline > $O/bench_llama2-7b_from_pristine.json 2>> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload llama3-8b --no-cpu-baseline > $O/bench_llama3-8b.json 2>> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload llama2-13b --no-cpu-baseline > $O/bench_llama2-13b.json 2>> $O/bench.err
{
for tp in 1 2 4 8; do timeout 300 python scripts/bench_shard.py llama2-7b --tp $tp --steps 20 2>&1 | tail -1; done
for tp in 2 4 8; do timeout 300 python scripts/bench_shard.py llama2-13b --tp $tp --steps 20 2>&1 | tail -1; done
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 2>&1 | tail -1
timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 --switch-mode from_pristine 2>&1 | tail -1
echo "# tp_push step of a shard timed alone (chained launches; the rank is its own and only peer: no NVLink traffic, no peers to wait for)"
for w in "llama2-7b --tp 8" "llama2-7b --tp 4" "llama2-13b --tp 8" "llama2-13b --tp 4"; do timeout 300 python scripts/bench_shard.py $w --steps 20 --push 2>&1 | tail -1; done
} > $O/tp_shard_alone.txt 2>&1
{
timeout 200 python scripts/bench_switch.py --config 7b --modes mma --iters 4 2>&1 | grep '"mode"'
timeout 200 python scripts/bench_switch.py --config 8b --modes mma --iters 4 2>&1 | grep '"mode"'
timeout 200 python scripts/bench_switch.py --config 13b --modes mma --iters 4 2>&1 | grep '"mode"'
for k in 1 2 4; do timeout 200 python scripts/bench_switch.py --config 70b-tp8 --layers 24 --k $k --modes mma --iters 4 2>&1 | grep '"mode"'; done
} > $O/switch_by_stacked_rank.txt 2>&1
{ timeout 200 python scripts/bench_attn.py --ctx 128 --splits 1,2,4; timeout 200 python scripts/bench_attn.py --ctx 1024 --splits 8,16,17,32; timeout 200 python scripts/bench_attn.py --ctx 4096 --splits 16,32;
  AF_ATTN2=0 timeout 200 python scripts/bench_attn.py --ctx 1024 --splits 8; } > $O/attn.txt 2>&1
{ for pc in 2 3; do AF_UMMA_PIECES=$pc timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('AF_UMMA_PIECES=$pc', 'ms_per_step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],2), 'tok/s; roofline frac', round(d['roofline']['frac'],4), d['roofline']['kernel'][:70])"; done
  for pc in 2 3; do echo "AF_UMMA_PIECES=$pc:"; AF_UMMA_PIECES=$pc timeout 600 python -m pytest tests/test_gpu_true_shapes.py -q -s -k "bench" 2>&1 | grep -E "elements checked|passed|failed" | cut -c1-330; done; } > $O/three_pieces.txt 2>&1
timeout 300 python scripts/timeline_chase.py --ctx 1024 --show 0,1,17,32 > $O/chase_timeline.txt 2>&1
timeout 200 ./scripts/micro/_bin/umma_rate > $O/umma_rate.txt 2>&1
if [ "$1" != "noncu" ]; then
AF_NCU=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
AF_NCU=1 timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:switch_umma -s 17 -c 1 -o $O/prof_chase -f \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_chase.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:switch_umma -s 3 -c 1 -o $O/prof_shard -f \
   python scripts/bench_shard.py llama2-7b --tp 4 --steps 2 > $O/ncu_shard.log 2>&1
fi
grep -E "passed|failed|error" $O/tests.log | head -40; tail -2 $O/smoke.log; cat $O/bench.json | cut -c1-600; tail -3 $O/bench.err; cat $O/tp_shard_alone.txt | cut -c1-200
tail -3 $O/ncu_launches.log $O/ncu_chase.log $O/ncu_shard.log 2>/dev/null | cut -c1-300
ls -la $O | head -50
