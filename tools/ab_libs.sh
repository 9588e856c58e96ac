#!/bin/bash
# Interleaved A/B of two builds of the library (abtmp/lib_a.so, abtmp/lib_b.so,
# copied there before the gpurun call).  Default measurement: the c3
# single-batch and pipelined steps of tools/pipe_bench.py; any other command
# can be given after the round count (its stdout is printed per run).
# usage (under gpurun): bash tools/ab_libs.sh [rounds] [command ...]
L=paper_2409_07704_b200/_lib/libmonoalign_b200.so
ROUNDS=${1:-3}
shift
for i in $(seq 1 $ROUNDS); do
  for v in a b; do
    cp abtmp/lib_$v.so $L
    if [ $# -gt 0 ]; then
      echo "$v $("$@" 2>&1 | tail -1)"
    else
      echo "$v $(python tools/pipe_bench.py 60 | grep -o '"plain": {"ms_per_step": [0-9.]*\|"pipelined": {"ms_per_step": [0-9.]*' | tr '\n' ' ')"
    fi
  done
done
