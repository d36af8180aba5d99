# parity + per-config profile + bench + ncu source-level capture of k_sim
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_sim.py > gpurun_out/prof_sim.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sim -c 1 -o gpurun_out/prof_sim python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sim.log 2>&1
