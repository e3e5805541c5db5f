#!/bin/bash
# attention planner: per-piece overhead in the range cutting (MTKV_ATTN_PIECE_COST, tiles): bars, micro, bench
set -u
O=gpurun_out/${1:-piece_cost}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_numerics.py -q -x -p no:cacheprovider -k "relative_bar or configs1" > $O/tests.log 2>&1
echo "exit $?" >> $O/tests.log
for c in 0 2 3 1.5 0; do
  MTKV_ATTN_PIECE_COST=$c timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 10 --tag pre_c$c >> $O/attn.jsonl 2>&1
  MTKV_ATTN_PIECE_COST=$c timeout 300 python tools/attn_bench.py --repeat 20 --tag dec_c$c >> $O/attn.jsonl 2>&1
done
for c in 0 2; do
  MTKV_ATTN_PIECE_COST=$c timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_c$c.json 2>/dev/null
done
