#!/bin/bash
# ncu evidence for the current build (run under gpurun): launch list of a
# short bench run and one full capture each of K1 (forward) and K2
# (backtrack) at BASELINE config 3.  usage: bash tools/profile.sh <tag>
TAG=${1:-dev}
O=gpurun_out
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd -s 2 -c 1 \
  -o $O/prof_fwd_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_fwd_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_walk -s 2 -c 1 \
  -o $O/prof_bt_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_bt_$TAG.log 2>&1
ls -la $O | grep $TAG
# K1g (fused log-likelihood) full capture
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd4 -s 1 -c 1 \
  -o $O/prof_fwdg_$TAG -f python tools/gauss_k1.py 80 > $O/ncu_fwdg_$TAG.log 2>&1
bash tools/l2_sequence.sh $TAG
