#!/bin/bash
# attention kernel A/B on tools/attn_bench.py (fixed synthetic batch, bench-layer shape)
timeout 300 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -s -k "attention" 2>&1 | grep -E "err|passed|failed" > gpurun_out/attn_ab_tests.log
for P in heads flat alt; do
  MTKV_ATTN_PART=$P timeout 120 python tools/attn_bench.py --tag part_$P >> gpurun_out/attn_ab.jsonl 2>&1
done
