#!/bin/bash
# one full ncu capture of the attention kernel on the microbenchmark batch
TAG=${1:-n}
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${TAG}_attn python tools/attn_bench.py --repeat 3 > gpurun_out/${TAG}_ncu.log 2>&1
