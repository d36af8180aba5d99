# round 2 session 3, first call: parity on a fresh box, phase profile of the 1,024 sweep, ncu
# source-level captures of k_sim (critical config alone; config 5 throughput variant)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scripts/build_variant.sh phases -DTWB_PROFILE_PHASES
TWB_PROF_STRIDE=32 TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_sim.py > gpurun_out/prof_phases.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim -c 1 -f -o gpurun_out/crit python scripts/prof_one.py 813 > gpurun_out/ncu_crit.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sim -c 1 -f -o gpurun_out/sim65k python scripts/ab_c5.py model 1 > gpurun_out/ncu_sim65k.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 30 gpurun_out/prof_phases.log
