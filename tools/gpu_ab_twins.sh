#!/bin/bash
# A/B of the twin (sibling-CTA) scheduling of 2-query-tile requests + dram bytes of one launch each.
NCU=/usr/local/cuda/bin/ncu
for T in 1 0; do
  MTKV_ATTN_TWINS=$T timeout 300 python bench.py --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/ab_twins$T.log 2>&1
  MTKV_ATTN_TWINS=$T timeout 600 $NCU --nvtx --nvtx-include "timed/" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:attn_tc_kernel -s 4 -c 2 --csv --log-file gpurun_out/ab_twins${T}_ncu.csv python bench.py --users 1024 --steps 6 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
done
