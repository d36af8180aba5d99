mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py -x -q -k "seg or sweep_1024 or small_cases or throughput or slot" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
for r in 1 2; do
  timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_mout.log 2>&1
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_old.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_mout.log 2>&1
done
timeout 300 python scripts/ab_env.py >> gpurun_out/ab_mout.log 2>&1
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_old.so timeout 300 python scripts/ab_env.py >> gpurun_out/ab_mout.log 2>&1
tail -n 2 gpurun_out/pytest_ab.log; cat gpurun_out/ab_mout.log
