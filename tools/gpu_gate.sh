#!/bin/bash
set -u
O=gpurun_out/${1:-gate}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_numerics.py tests/test_gpu_engine.py -q -x -p no:cacheprovider > $O/tests.log 2>&1
echo "pytest exit $?" >> $O/tests.log
timeout 300 python tools/kernel_times.py --steps 8 --warm 30 > $O/kt.jsonl 2>/dev/null
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gate_block_kernel -c 3 --csv python tools/kernel_times.py --steps 1 --warm 30 --ncu --policy adaptive > $O/gate_ncu.csv 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench.json 2>/dev/null
