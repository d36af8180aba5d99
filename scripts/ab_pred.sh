mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do for v in bucket bucket4 rcp5; do
  TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so python scripts/ab_pred.py 2>/dev/null | sed "s/^/$v: /" >> gpurun_out/ab_pred.log
done; done
