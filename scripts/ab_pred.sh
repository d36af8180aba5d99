# A/B bulk-predictor variants (built by scripts/build_variant.sh) on one box: tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do for v in $AB_VARIANTS; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/ab_pred.py 2>/dev/null | sed "s/^/$v: /" >> gpurun_out/ab_pred.log
done; done
