#!/bin/bash
# Quick GPU iteration: GPU tests + bench (no ncu).
TAG=${1:-q}
timeout 600 python -m pytest tests -q -m gpu -s -x 2>&1 | grep -E "rel logit|err|passed|failed|Error|assert" > gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
