#!/bin/bash
timeout 200 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -k "attention" 2>&1 | tail -1 > gpurun_out/v3b_tests.log
timeout 120 python tools/attn_bench.py --tag v3_nk3 > gpurun_out/v3b_attn.jsonl 2>&1
timeout 120 python tools/attn_bench.py --tail-frac 0 --tag v3_nk3_notail >> gpurun_out/v3b_attn.jsonl 2>&1
