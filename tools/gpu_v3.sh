#!/bin/bash
timeout 200 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -s -k "attention or bench_config or value_engine" 2>&1 | grep -E "err|passed|failed|Error|assert" > gpurun_out/v3_tests.log
timeout 120 python tools/attn_bench.py --tag v3 > gpurun_out/v3_attn.jsonl 2>&1
timeout 120 python tools/attn_bench.py --tail-frac 0 --tag v3_notail >> gpurun_out/v3_attn.jsonl 2>&1
