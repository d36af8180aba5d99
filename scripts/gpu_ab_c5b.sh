mkdir -p gpurun_out; rm -f gpurun_out/ab_c5b.log
for r in 1 2; do
for lib in olddig base vb; do
  L=paper_2601_00397_b200/lib/libtwb200_$lib.so
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=$L timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_c5b.log 2>&1
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=$L timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_c5b.log 2>&1
done
done
for lib in olddig base vb; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_sample_count,gpu__time_duration.sum --clock-control none -k regex:k_sim -c 1 python scripts/ab_c5.py model 1 > gpurun_out/ncu_c5_$lib.log 2>&1
  grep -E "inst_executed|issue_active|no_instr|sample_count|duration" gpurun_out/ncu_c5_$lib.log | sed "s/^/$lib /" >> gpurun_out/ab_c5b.log
done
cat gpurun_out/ab_c5b.log
