L=paper_2409_07704_b200/_lib/libmonoalign_b200.so
python tools/ab.py 32 1024 8192 $L build/var_pn.so build/var_pu.so build/var_nn.so > gpurun_out/ab_pol.txt 2>&1
for v in $L build/var_pn.so build/var_pu.so; do
  MAS_LIB_PATH=$v timeout 300 ncu --cache-control none --clock-control none -k regex:mas_fwd4 -s 2 -c 1 --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv python tools/prof_run.py 32 1024 8192 3 2>/dev/null | grep -E "dram|duration" | sed "s|^|$v |" >> gpurun_out/ab_pol_ncu.txt
done
