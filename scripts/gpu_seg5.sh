mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -x -q -k "seg or sweep_1024 or small_cases or timekeeper" > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 600 python scripts/seg_stats.py 0 8 16 32 > gpurun_out/seg_stats.log 2>&1
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_no_instructions
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv python scripts/seg_one.py config4 16 > gpurun_out/seg_config4_16.csv 2>&1
tail -n 3 gpurun_out/pytest_seg.log; cat gpurun_out/seg_stats.log
