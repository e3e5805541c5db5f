#!/bin/bash
timeout 200 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -k "attention" 2>&1 | tail -1 > gpurun_out/ab3_tests.log
for P in 8 4 0; do MTKV_ATTN_POLY=$P timeout 120 python tools/attn_bench.py --tag poly$P >> gpurun_out/ab3.jsonl 2>&1; done
for P in 8 0; do MTKV_ATTN_POLY=$P timeout 120 python tools/attn_bench.py --tail-frac 0 --tag notail_poly$P >> gpurun_out/ab3.jsonl 2>&1; done
