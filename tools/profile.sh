#!/bin/bash
# ncu evidence for the current build (run under gpurun; outputs in
# gpurun_out/, summarised into profiles/ by tools/ncu_summary.py):
#   launch list of a short bench run (gpu__time_duration per launch),
#   full captures of K1 (forward), K2 (backtrack), K1g (fused Gaussian),
#   K1s (score export), the GaussianPlan launch list, the K1 -> K2 L2
#   sequence, and K1's per-instruction stall samples.
# usage: bash tools/profile.sh <tag>
TAG=${1:-dev}
O=gpurun_out
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd -s 2 -c 1 \
  -o $O/prof_fwd_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_fwd_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_walk -s 2 -c 1 \
  -o $O/prof_bt_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_bt_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd4 -s 1 -c 1 \
  -o $O/prof_fwdg_$TAG -f python tools/gauss_k1.py 80 > $O/ncu_fwdg_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd4 -s 1 -c 1 \
  -o $O/prof_scores_$TAG -f python tools/scores_run.py 3 > $O/ncu_scores_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_gauss_$TAG.csv python tools/gauss_plan_run.py 80 3 \
  > /dev/null 2>&1
ncu -i $O/prof_fwd_$TAG.ncu-rep --page source --csv --print-source sass > $O/fwd_${TAG}_source.csv 2>&1
bash tools/l2_sequence.sh $TAG
ls -la $O | grep $TAG
