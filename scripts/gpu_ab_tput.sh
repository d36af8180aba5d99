mkdir -p gpurun_out; rm -f gpurun_out/ab_tput.log
V=${AB_VARIANTS:-"vb tpred ttk tcold2 tall olddig"}
for r in 1 2; do
for lib in $V; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_tput.log 2>&1
done
done
for lib in $V; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model1k 5 >> gpurun_out/ab_tput.log 2>&1
done
cat gpurun_out/ab_tput.log
