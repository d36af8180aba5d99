mkdir -p gpurun_out
timeout 600 python scripts/ab_env.py "TWB_SIM_SEG_LAT=1" "TWB_SIM_SEG_LAT=1 TWB_SIM_SEG_STAGE=33056" "TWB_SIM_SEG_W=12" > gpurun_out/ab_env.log 2>&1
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_inl.so timeout 600 python scripts/ab_env.py > gpurun_out/ab_env_inl.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim_seg -s 1 -c 1 -f -o gpurun_out/seg4 python scripts/seg_one.py config4 16 > gpurun_out/ncu_seg4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_seg_tk -s 1 -c 1 -f -o gpurun_out/segtk4 python scripts/seg_one.py config4 16 > gpurun_out/ncu_segtk4.log 2>&1
cat gpurun_out/ab_env.log gpurun_out/ab_env_inl.log
