mkdir -p gpurun_out; rm -f gpurun_out/ab_ext.log
for i in 1 2; do for v in e0 ec euc; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/ab_ext.py 2>/dev/null | sed "s/^/$v: /" >> gpurun_out/ab_ext.log
done; done
for v in ec; do
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_extraction or csr or larger_than" 2>&1 | tail -1 | sed "s/^/$v parity: /" >> gpurun_out/ab_ext.log
done
cat gpurun_out/ab_ext.log
