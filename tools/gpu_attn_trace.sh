#!/bin/bash
TAG=${1:-t}
MTKV_ATTN_TRACE=gpurun_out/attn_${TAG}.bin timeout 120 python tools/attn_bench.py --repeat 5 --tag $TAG > gpurun_out/attn_${TAG}.json 2>&1
python tools/attn_trace.py gpurun_out/attn_${TAG}.bin 3 > gpurun_out/attn_${TAG}.txt 2>&1
timeout 120 python tools/attn_bench.py --tag ${TAG}_untraced >> gpurun_out/attn_${TAG}.json 2>&1
