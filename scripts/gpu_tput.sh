# GPU suite with the two k_sim variants, then old (core-staged) vs new at 65,536 and 1,024 configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
rm -f gpurun_out/ab_tput.log
for i in 1 2; do
  STAGE=core TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_old.so timeout 600 python scripts/ab_65k.py 2>/dev/null | sed "s/^/old 65k: /" >> gpurun_out/ab_tput.log
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_new.so timeout 600 python scripts/ab_65k.py 2>/dev/null | sed "s/^/new 65k: /" >> gpurun_out/ab_tput.log
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_old.so timeout 300 python scripts/prof_sim.py 2>/dev/null | head -1 | sed "s/^/old 1k: /" >> gpurun_out/ab_tput.log
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_new.so timeout 300 python scripts/prof_sim.py 2>/dev/null | head -1 | sed "s/^/new 1k: /" >> gpurun_out/ab_tput.log
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/ab_tput.log
