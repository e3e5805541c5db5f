#!/bin/bash
# deferred attention epilogue: bars (watchdog build), then timing build micro (prefill / decode) + trace
set -u
O=gpurun_out/${1:-epi}
mkdir -p $O
MTKV_NVCC_EXTRA=-DMTKV_WATCHDOG timeout 600 python -m paper_2604_22881_b200.build --force > $O/build_wd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_numerics.py -q -x -p no:cacheprovider > $O/tests_wd.log 2>&1
rc=$?
echo "pytest exit $rc" >> $O/tests_wd.log
[ $rc -eq 0 ] || exit 1
timeout 600 python -m paper_2604_22881_b200.build --force > $O/build.log 2>&1
for i in 1 2; do
  timeout 300 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 10 --tag pre >> $O/attn.jsonl 2>&1
  timeout 300 python tools/attn_bench.py --repeat 20 --tag dec >> $O/attn.jsonl 2>&1
done
MTKV_ATTN_TRACE=$O/pre.bin timeout 120 python tools/attn_bench.py --requests 24 --prefix 0 --nq 4096 --tail-frac 0 --repeat 3 > /dev/null 2>&1
python tools/attn_trace_stats.py $O/pre.bin > $O/pre.txt 2>&1
