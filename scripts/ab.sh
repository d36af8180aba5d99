# A/B the k_sim variants on the same box (alternating runs)
mkdir -p gpurun_out
for i in 1 2; do
  for v in $AB_VARIANTS; do
    TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/prof_sim.py 2>/dev/null | head -1 | sed "s/^/$v: /" >> gpurun_out/ab.log
  done
done
