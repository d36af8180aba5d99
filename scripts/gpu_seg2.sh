mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py -x -q > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for a in "config4 16" "config4 8" "config3 32" "config1 0"; do
  set -- $a
  timeout 300 ncu --metrics $M --clock-control none --csv python scripts/seg_one.py $1 $2 > gpurun_out/seg_$1_$2.csv 2>&1
done
tail -n 5 gpurun_out/pytest_seg.log
