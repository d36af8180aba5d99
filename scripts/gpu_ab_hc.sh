mkdir -p gpurun_out; rm -f gpurun_out/ab_hc.log
for r in 1 2; do for lib in h0 hc; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_hc.log 2>&1
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_hc.log 2>&1
done; done
timeout 600 python scripts/ab_e2e65.py >> gpurun_out/ab_hc.log 2>&1
cat gpurun_out/ab_hc.log
