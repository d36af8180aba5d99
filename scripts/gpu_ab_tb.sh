mkdir -p gpurun_out; rm -f gpurun_out/ab_tb.log
timeout 600 python scripts/ab_e2e65.py >> gpurun_out/ab_tb.log 2>&1
for r in 1 2; do for lib in tb4 tb5 tb6; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_tb.log 2>&1
done; done
cat gpurun_out/ab_tb.log
