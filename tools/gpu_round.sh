#!/bin/bash
# One GPU session: parity tests, smoke, bench (default), launch list of the
# timed phase + one full ncu capture of the attention kernel in the timed phase.
# Outputs under gpurun_out/<tag>_*.
set -x
TAG=${1:-r01}
python -m pytest tests -q -m gpu -s 2>&1 | grep -E "rel logit|err|passed|failed|Error" > gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
NCU=/usr/local/cuda/bin/ncu
PROF_ARGS=${PROF_ARGS:-"--users 1024 --steps 6 --warmup 4 --no-cpu-baseline"}
timeout 900 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py ${PROF_ARGS} > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
   -k regex:attn_tc_kernel -s 4 -c 1 -o gpurun_out/${TAG}_attn python bench.py ${PROF_ARGS} \
   > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
