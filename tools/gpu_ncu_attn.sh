#!/bin/bash
# Full ncu capture of one attn_tc_kernel launch inside the timed phase.
TAG=${1:-n}
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
   -k regex:attn_tc_kernel -s 4 -c 1 -o gpurun_out/${TAG}_attn python bench.py --users 1024 --steps 6 --warmup 4 --no-cpu-baseline \
   > gpurun_out/${TAG}_ncu_full.log 2>&1
