mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for v in "" tk5 tk8; do
  if [ -n "$v" ]; then export TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so; fi
  timeout 300 ncu --metrics $M --clock-control none --csv -k regex:k_seg_tk python scripts/seg_one.py config4 > gpurun_out/segtk_$v.csv 2>&1
  timeout 300 python scripts/ab_env.py > gpurun_out/ab_tk_$v.log 2>&1
done
for v in "" tk5 tk8; do echo "== $v"; cat gpurun_out/ab_tk_$v.log; grep -h "gpu__time_duration" gpurun_out/segtk_$v.csv | tail -1; done
