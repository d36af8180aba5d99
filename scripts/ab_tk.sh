mkdir -p gpurun_out; rm -f gpurun_out/ab_tk.log
for v in $AB_VARIANTS; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/ab_tk.py 2>&1 | tail -1 | sed "s/^/$v: /" >> gpurun_out/ab_tk.log
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "tk" 2>&1 | tail -1 | sed "s/^/$v tests: /" >> gpurun_out/ab_tk.log
done
