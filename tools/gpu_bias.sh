#!/bin/bash
# adaptive policy: bias on the calibrated layer-stack rate (more / less re-encoding), bench lines
set -u
O=gpurun_out/${1:-bias}
mkdir -p $O
for b in 1.0 1.2 1.4 0.85 1.0; do
  MTKV_ADAPTIVE_SM_BIAS=$b timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/bench_b$b.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/bench_b$b.json'));print('$b', round(d['value']), round(d['e2e']['value']), d['phases']['A_device']['prefix_recomputed_frac'], round(d['host_link']['frac'],3), d['clocks']['sm_mhz'])" >> $O/summary.txt
done
