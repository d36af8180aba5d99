# critical-config evidence: phase profile (TWB_PROFILE_PHASES build) of the 1,024 sweep, and ncu
# source-level capture of config 45 alone (per-SASS-line instruction counts and stall samples)
mkdir -p gpurun_out
bash scripts/build_variant.sh phases -DTWB_PROFILE_PHASES
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_sim.py > gpurun_out/prof_phases.log 2>&1
timeout 300 python scripts/prof_one.py 45 > gpurun_out/prof_one.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim -c 1 -f -o gpurun_out/crit45 python scripts/prof_one.py 45 > gpurun_out/ncu_crit.log 2>&1
echo done
