#!/bin/bash
# paired kernel (MTKV_ATTN_PAIR=1): watchdog build + bars, then timing build: traced prefill, prefill / decode vs one-tile
set -u
O=gpurun_out/${1:-attn_pair}
mkdir -p $O
export MTKV_ATTN_PAIR=1
MTKV_NVCC_EXTRA=-DMTKV_WATCHDOG timeout 600 python -m paper_2604_22881_b200.build --force > $O/build_wd.log 2>&1
timeout 300 python -m pytest tests/test_gpu_numerics.py -q -x -s -p no:cacheprovider -k "relative_bar and -128-" > $O/tests_wd.log 2>&1
rc=$?
echo "pytest exit $rc" >> $O/tests_wd.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m paper_2604_22881_b200.build --force > $O/build.log 2>&1
MTKV_ATTN_TRACE=$O/pre.bin timeout 120 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 3 > /dev/null 2>&1
python tools/attn_trace_stats.py $O/pre.bin > $O/pre.txt 2>&1
for p in 1 0; do
  MTKV_ATTN_PAIR=$p timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 20 --tag pre_pair$p >> $O/attn.jsonl 2>&1
  MTKV_ATTN_PAIR=$p timeout 300 python tools/attn_bench.py --repeat 20 --tag dec_pair$p >> $O/attn.jsonl 2>&1
done
