mkdir -p gpurun_out; rm -f gpurun_out/ab_c5.log
for r in 1 2; do
for lib in olddig default; do
  for k in old model; do
    if [ $lib = default ]; then L=paper_2601_00397_b200/lib/libtwb200.so; else L=paper_2601_00397_b200/lib/libtwb200_$lib.so; fi
    TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=$L timeout 300 python scripts/ab_c5.py $k 3 >> gpurun_out/ab_c5.log 2>&1
  done
done
done
for lib in olddig default; do
  if [ $lib = default ]; then L=paper_2601_00397_b200/lib/libtwb200.so; else L=paper_2601_00397_b200/lib/libtwb200_$lib.so; fi
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=$L timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_c5.log 2>&1
done
cat gpurun_out/ab_c5.log
