#!/bin/bash
# one-tile attention: L2 prefetch cursor depth (MTKV_ATTN_PREFETCH), decode / prefill microbenchmarks, bench phase B roofline
set -u
O=gpurun_out/${1:-pf}
mkdir -p $O
MTKV_ATTN_PREFETCH=4 timeout 300 python -m pytest tests/test_gpu_numerics.py -q -x -p no:cacheprovider -k "relative_bar" > $O/tests_pf4.log 2>&1
echo "exit $?" >> $O/tests_pf4.log
for p in 0 2 4 8 0; do
  MTKV_ATTN_PREFETCH=$p timeout 300 python tools/attn_bench.py --repeat 20 --tag dec_pf$p >> $O/attn.jsonl 2>&1
  MTKV_ATTN_PREFETCH=$p timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 10 --tag pre_pf$p >> $O/attn.jsonl 2>&1
done
for p in 0 4; do
  MTKV_ATTN_PREFETCH=$p timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_pf$p.json 2>/dev/null
done
