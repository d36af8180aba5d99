# round-2 session-2 probes: phase mix of configs 4/5 (TWB_PROFILE_PHASES build), extraction back-off A/B
mkdir -p gpurun_out
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 600 python scripts/prof_iters65.py > gpurun_out/iters65.log 2>&1
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_iters65.py 1024 > gpurun_out/iters1k.log 2>&1
TWB_PROF_STRIDE=32 TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_sim.py > gpurun_out/prof_phases1k.log 2>&1
AB_VARIANTS="bo0 bo64 bo256 bo1000" bash scripts/ab_ext2.sh
cat gpurun_out/iters65.log gpurun_out/iters1k.log
