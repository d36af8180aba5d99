mkdir -p gpurun_out; rm -f gpurun_out/ab_r2d.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "beyond or linear_quant or zero_and_negative" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
tail -n 2 gpurun_out/pytest_new.log >> gpurun_out/ab_r2d.log
for r in 1 2 3; do
for lib in v0 rcp cm rcpcm; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_r2d.log 2>&1
done
done
for lib in v0 rcpcm; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_r2d.log 2>&1
done
cat gpurun_out/ab_r2d.log
