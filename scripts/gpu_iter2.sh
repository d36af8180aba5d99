mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_phases.so timeout 300 python scripts/prof_sim.py > gpurun_out/prof_sim.log 2>&1
timeout 300 python scripts/prof_sim.py 2>/dev/null | head -1 > gpurun_out/prof_plain.log
python scripts/prof_one.py 24 > gpurun_out/prof_one.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
