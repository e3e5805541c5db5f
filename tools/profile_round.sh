#!/bin/bash
# One GPU pass of the round's evidence (run under gpurun from the repo root):
#   tools/profile_round.sh <tag>
# -> gpurun_out/<tag>_{gpu_tests.log,smoke.log,bench.json,launches_*.csv,*_ncu.ncu-rep}
set -u
T=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rs -p no:cacheprovider --durations=15 > $O/${T}_gpu_tests.log 2>&1
echo "pytest exit $?" >> $O/${T}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
# per-kernel device time of 4 steady-state batches, both host-hit policies (serialised, cold caches: shares)
for pol in always adaptive; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${T}_launches_${pol}.csv python tools/kernel_times.py --steps 4 --warm 30 --ncu --policy $pol > /dev/null 2>&1
done
# full captures: attention on a decode batch, the projection GEMM and gate/norm on an adaptive batch
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tc_kernel -c 1 \
  -o $O/${T}_attn_ncu python tools/kernel_times.py --steps 1 --warm 30 --ncu --policy always > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_ps_kernel -c 1 \
  -o $O/${T}_gemm_ncu python tools/kernel_times.py --steps 1 --warm 30 --ncu --policy adaptive > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:gate_block_kernel -c 1 \
  -o $O/${T}_gate_ncu python tools/kernel_times.py --steps 1 --warm 30 --ncu --policy adaptive > /dev/null 2>&1
ls -la $O | grep $T
# the other BASELINE configs and the reference arm (bench lines)
bash tools/configs_sweep.sh $T
for c in gr8_d512 tiny_d64; do
  timeout 900 python bench.py --no-cpu-baseline --steps 20 --config $c 2>/dev/null | tail -1 > $O/${T}_bench_$c.json
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_reference_arm.json 2>&1
python tools/planner_scale.py --batches 30 > $O/${T}_planner_scale.jsonl 2>/dev/null
ls -la $O | grep $T
