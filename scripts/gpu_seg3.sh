mkdir -p gpurun_out
timeout 600 python scripts/seg_stats.py 0 16 32 64 > gpurun_out/seg_stats.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim_seg -s 1 -c 1 -f -o gpurun_out/seg4 python scripts/seg_one.py config4 16 > gpurun_out/ncu_seg4.log 2>&1
cat gpurun_out/seg_stats.log
