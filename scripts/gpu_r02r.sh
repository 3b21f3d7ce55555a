#!/bin/bash
O=gpurun_out
rm -f $O/tests_final.log
for f in tests/test_gpu_*.py tests/test_harness.py tests/test_io.py; do
  echo "=== $f" >> $O/tests_final.log
  timeout 1500 python -m pytest $f -q -m gpu -s --timeout 1200 --timeout-method=thread 2>&1 | grep -vE "^$" | cut -c1-400 | tail -14 >> $O/tests_final.log
done
timeout 300 python __graft_entry__.py smoke > $O/smoke_final.log 2>&1; echo "exit $?" >> $O/smoke_final.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_final.json 2> $O/bench_final.err
{ timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 2>&1 | tail -1; timeout 300 python scripts/bench_shard.py llama2-70b --tp 8 --steps 10 --switch-mode from_pristine 2>&1 | tail -1; } > $O/tp_shard_70b_final.txt
grep -E "===|passed|failed" $O/tests_final.log; tail -2 $O/smoke_final.log; cut -c1-300 $O/bench_final.json; cat $O/tp_shard_70b_final.txt | cut -c1-200
