#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -s -k "attention or value_engine or bench_config" 2>&1 | grep -E "passed|failed|Error" > gpurun_out/pdl_tests.log
timeout 120 python tools/attn_bench.py --tag pdl > gpurun_out/pdl_attn.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/pdl_bench.log 2>&1
