#!/bin/bash
for tf in 0.69 0.0; do timeout 120 python tools/attn_bench.py --tail-frac $tf --tag tail$tf >> gpurun_out/ab2.jsonl 2>&1; done
