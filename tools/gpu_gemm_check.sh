#!/bin/bash
timeout 400 python -m pytest tests -q -m gpu -x -s 2>&1 | grep -E "rel logit|err|passed|failed|Error|assert" > gpurun_out/g1_tests.log
MTKV_GEMM=mma timeout 200 python tools/ab_attention.py > /dev/null 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/g1_launches.csv python bench.py --users 1024 --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/g1_ncu_bench.log 2>&1
