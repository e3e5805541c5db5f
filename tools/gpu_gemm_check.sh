#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -k "value_engine or bench_config" 2>&1 | tail -1 > gpurun_out/g2_tests.log
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/g2_launches.csv python bench.py --users 1024 --steps 6 --warmup 4 --no-cpu-baseline > gpurun_out/g2_ncu_bench.log 2>&1
timeout 600 python tools/sweep.py ablation > gpurun_out/sweep_ablation.jsonl 2> gpurun_out/sweep_ablation.err
