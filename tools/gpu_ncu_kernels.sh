#!/bin/bash
# Full ncu captures of the non-attention kernels of one bench step (timed NVTX range):
# projection GEMM + fused KV append, the two MLP GEMMs, gate_norm.
TAG=${1:-k}
NCU=/usr/local/cuda/bin/ncu
ARGS="--users 1024 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
   -k regex:gemm_tc_kernel -c 3 -o gpurun_out/${TAG}_gemm python bench.py $ARGS > gpurun_out/${TAG}_ncu_gemm.log 2>&1
timeout 600 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
   -k regex:gate_norm -c 1 -o gpurun_out/${TAG}_gate python bench.py $ARGS > gpurun_out/${TAG}_ncu_gate.log 2>&1
ls -la gpurun_out | grep ${TAG}_
