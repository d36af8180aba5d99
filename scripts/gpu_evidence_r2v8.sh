# round-2 v8 evidence (end of session 4): tests, smoke, bench, ncu of the summary kernels, and the
# four compute-sanitizer tools over every kernel (the summary kernel changed in session 4)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_metrics -s 2 -c 2 -f -o gpurun_out/prof_metrics python scripts/ab_metrics.py 65536 > gpurun_out/ncu_metrics.log 2>&1
bash scripts/sanitize.sh > gpurun_out/sanitize_summary.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/sanitize_summary.log; tail -c 300 gpurun_out/bench.log
