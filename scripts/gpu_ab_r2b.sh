mkdir -p gpurun_out; rm -f gpurun_out/ab_r2b.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sim or sweep" > gpurun_out/pytest_sim.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sim.log
tail -n 2 gpurun_out/pytest_sim.log >> gpurun_out/ab_r2b.log
for r in 1 2; do
for lib in p1 p2 p3 p4; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_r2b.log 2>&1
done
for lib in p1 l1; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_r2b.log 2>&1
done
done
cat gpurun_out/ab_r2b.log
