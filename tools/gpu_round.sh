#!/bin/bash
# One GPU session: parity tests, bench (default), launch list + one full ncu
# capture of the attention kernel. Outputs under gpurun_out/.
set -x
TAG=${1:-r01}
python -m pytest tests -q -m gpu -s 2>&1 | grep -E "rel logit|err|passed|failed|Error" > gpurun_out/${TAG}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --users 256 --steps 4 --warmup 3 --no-cpu-baseline \
   > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 40 -c 2 \
   -o gpurun_out/${TAG}_attn python bench.py --users 256 --steps 4 --warmup 3 --no-cpu-baseline \
   > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
