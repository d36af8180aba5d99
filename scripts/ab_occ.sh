# A/B k_sim variants at both regimes (65,536 and 1,024 configs), alternating rounds
mkdir -p gpurun_out; rm -f gpurun_out/ab_occ.log
for i in 1 2; do for v in $AB_VARIANTS; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 600 python scripts/ab_65k.py 2>/dev/null | sed "s/^/$v 65k: /" >> gpurun_out/ab_occ.log
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/prof_sim.py 2>/dev/null | head -1 | sed "s/^/$v 1k: /" >> gpurun_out/ab_occ.log
done; done
cat gpurun_out/ab_occ.log
