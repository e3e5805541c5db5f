#!/bin/bash
# pair kernel timing only (no rebuild): traced prefill, untraced prefill / decode, both kernels
set -u
O=gpurun_out/${1:-pair3}
mkdir -p $O
MTKV_ATTN_TRACE=$O/pre.bin timeout 120 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 3 > $O/pre_traced.log 2>&1
python tools/attn_trace_stats.py $O/pre.bin > $O/pre.txt 2>&1
for p in 1 0; do
  MTKV_ATTN_PAIR=$p timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 20 > $O/prefill_pair$p.log 2>&1
  MTKV_ATTN_PAIR=$p timeout 300 python tools/attn_bench.py --repeat 20 > $O/decode_pair$p.log 2>&1
done
