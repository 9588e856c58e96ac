#!/bin/bash
# Source-level (SASS) stall samples of K1 at c3: one full ncu capture and
# its per-instruction CSV.  usage (under gpurun): bash tools/ncu_source.sh <tag>
TAG=${1:-dev}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd4 -s 2 -c 1 \
  -o $O/prof_fwd_$TAG -f python tools/prof_run.py 32 1024 8192 3 > $O/ncu_fwd_$TAG.log 2>&1
ncu -i $O/prof_fwd_$TAG.ncu-rep --page source --csv --print-source sass > $O/fwd_${TAG}_source.csv 2>&1
