#!/bin/bash
# BASELINE configs[2] (cache disabled / HBM only / hierarchical) and configs[4]
# (HBM pool 1-50 % of the working set) as bench.py lines (N = 1):
#   tools/configs_sweep.sh <tag>  ->  gpurun_out/<tag>_configs2.jsonl, <tag>_configs4.jsonl
T=${1:-r02}
O=gpurun_out
mkdir -p $O
: > $O/${T}_configs2.jsonl
for m in recompute gpu_only hierarchical; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --mode $m 2>/dev/null | tail -1 >> $O/${T}_configs2.jsonl
done
: > $O/${T}_configs4.jsonl
for f in 0.01 0.02 0.05 0.1 0.2 0.5; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --pool-frac $f 2>/dev/null | tail -1 >> $O/${T}_configs4.jsonl
done
wc -l $O/${T}_configs*.jsonl
