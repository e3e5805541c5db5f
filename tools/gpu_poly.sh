#!/bin/bash
# one-tile attention: exponentials partly on the FMA pipe (MTKV_ATTN_POLY=k: every k-th column), prefill and decode
set -u
O=gpurun_out/${1:-poly}
mkdir -p $O
for p in 0 8 4 3 2; do
  MTKV_ATTN_POLY=$p timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 20 --tag pre_poly$p >> $O/attn.jsonl 2>&1
  MTKV_ATTN_POLY=$p timeout 300 python tools/attn_bench.py --repeat 20 --tag dec_poly$p >> $O/attn.jsonl 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --e2e-depth 5 > $O/bench.json 2> $O/bench.err
