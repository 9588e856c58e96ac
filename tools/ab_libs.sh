#!/bin/bash
# Interleaved A/B of two builds of the library (abtmp/lib_a.so, abtmp/lib_b.so,
# copied there before the gpurun call) on tools/pipe_bench.py.
# usage (under gpurun): bash tools/ab_libs.sh [rounds]
L=paper_2409_07704_b200/_lib/libmonoalign_b200.so
for i in $(seq 1 ${1:-3}); do
  for v in a b; do
    cp abtmp/lib_$v.so $L
    echo "$v $(python tools/pipe_bench.py 60 | grep -o '"plain": {"ms_per_step": [0-9.]*\|"pipelined": {"ms_per_step": [0-9.]*' | tr '\n' ' ')"
  done
done
