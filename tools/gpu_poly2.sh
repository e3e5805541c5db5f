#!/bin/bash
set -u
O=gpurun_out/${1:-poly2}
mkdir -p $O
for p in 0 4 3 2; do
  MTKV_ATTN_PAIR=1 MTKV_ATTN_POLY=$p timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 20 --tag pair_pre_poly$p >> $O/attn.jsonl 2>&1
done
MTKV_ATTN_PAIR=1 MTKV_ATTN_POLY=2 timeout 300 python -m pytest tests/test_gpu_numerics.py -q -x -p no:cacheprovider -k "relative_bar and -128-" > $O/tests_poly2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --e2e-depth 5 > $O/bench.json 2> $O/bench.err
