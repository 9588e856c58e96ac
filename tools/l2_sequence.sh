#!/bin/bash
# K1 -> K2 as they run in the step, caches NOT flushed between kernels
# (--cache-control none) and the application replayed per metric pass, so
# K2's L2 hit rate on the direction words is the one it sees after K1
# (north-star evidence).  Run under gpurun:  bash tools/l2_sequence.sh <tag>
TAG=${1:-dev}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --cache-control none --clock-control none --replay-mode application \
  -k regex:"mas_fwd4|bt_walk" -s 4 -c 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_read_hit_rate.pct,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,smsp__pcsamp_warps_issue_stalled_branch_resolving,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_sample_count \
  --csv --log-file $O/l2seq_$TAG.csv python tools/prof_run.py 32 1024 8192 4 > $O/l2seq_$TAG.log 2>&1
