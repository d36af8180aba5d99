mkdir -p gpurun_out; rm -f gpurun_out/ab_ext.log
for i in 1 2; do for v in e0 epair enp epairnp; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 300 python scripts/ab_ext.py 2>/dev/null | sed "s/^/$v: /" >> gpurun_out/ab_ext.log
done; done
TWB_PROF_STRIDE=32 TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_sim.py > gpurun_out/prof_phases.log 2>&1
cat gpurun_out/ab_ext.log; head -6 gpurun_out/prof_phases.log; tail -4 gpurun_out/prof_phases.log
