mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -x -q -k "seg or sweep_1024 or small_cases or timekeeper" > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 600 python scripts/seg_stats.py 0 8 16 32 > gpurun_out/seg_stats.log 2>&1
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_segnoinl.so timeout 600 python scripts/seg_stats.py 0 16 > gpurun_out/seg_stats_noinl.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim_seg -s 1 -c 1 -f -o gpurun_out/seg4 python scripts/seg_one.py config4 16 > gpurun_out/ncu_seg4.log 2>&1
tail -n 3 gpurun_out/pytest_seg.log; cat gpurun_out/seg_stats.log gpurun_out/seg_stats_noinl.log
