mkdir -p gpurun_out; rm -f gpurun_out/ab_65only.log
for i in 1 2; do for v in $AB_VARIANTS; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 600 python scripts/ab_65k.py 2>/dev/null | sed "s/^/$v 65k: /" >> gpurun_out/ab_65only.log
done; done
cat gpurun_out/ab_65only.log
