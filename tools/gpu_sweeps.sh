#!/bin/bash
# configs[4] pressure sweep and configs[3] (8-layer d=512, 8K histories) per-GPU shard
timeout 900 python tools/sweep.py pressure > gpurun_out/sweep_pressure.jsonl 2> gpurun_out/sweep_pressure.err
timeout 600 python bench.py --config gr8_d512 --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/bench_gr8.log 2>&1
free -g > gpurun_out/box_mem.txt
