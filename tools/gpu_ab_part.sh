#!/bin/bash
# A/B of the attention work partitions (MTKV_ATTN_PART) on the bench layer (1024 users per GPU).
timeout 300 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -k "attention or bench_config" 2>&1 | tail -1 > gpurun_out/ab_part_tests.log
for P in heads alt flat; do
  MTKV_ATTN_PART=$P timeout 240 python bench.py --users 1024 --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/ab_part_$P.log 2>&1
done
