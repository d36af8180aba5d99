mkdir -p gpurun_out
bash scripts/sanitize.sh > gpurun_out/sanitize_summary.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/sanitize_summary.log; tail -n 3 gpurun_out/pytest_gpu.log
