#!/bin/bash
# persistent GEMM: silu partly on the FMA pipe (MTKV_GEMM_SILU_FMA=k): dense-op bars, in-situ kernel times, bench
set -u
O=gpurun_out/${1:-silu}
mkdir -p $O
for k in 2 4; do
  MTKV_GEMM_SILU_FMA=$k timeout 300 python -m pytest tests/test_gpu_engine.py -q -x -s -p no:cacheprovider -k "dense_op" > $O/tests_fma$k.log 2>&1
  echo "exit $?" >> $O/tests_fma$k.log
done
for k in 0 2 4 8; do
  MTKV_GEMM_SILU_FMA=$k timeout 300 python tools/kernel_times.py --steps 8 --warm 30 > $O/kt_fma$k.jsonl 2>/dev/null
done
for k in 0 4; do
  MTKV_GEMM_SILU_FMA=$k timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_fma$k.json 2>/dev/null
done
