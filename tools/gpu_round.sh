#!/bin/bash
# One GPU-box pass: parity tests, smoke, both bench arms, ncu launch list and
# a full capture of the forward kernel.  Outputs land in gpurun_out/.
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 600 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mas_fwd -s 2 -c 1 \
  -o $O/prof_fwd_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_fwd_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_walk -s 2 -c 1 \
  -o $O/prof_bt_$TAG -f python tools/prof_run.py 32 1024 8192 4 > $O/ncu_bt_$TAG.log 2>&1
tail -3 $O/pytest_gpu_$TAG.log; tail -2 $O/smoke_$TAG.log; cat $O/bench_$TAG.json $O/bench_ref_$TAG.json; tail -3 $O/bench_$TAG.err
