# predictor iteration: parity tests, bench line, ncu --set full of the bulk predictor
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_predict_features -s 2 -c 1 -o gpurun_out/prof_pred python scripts/ab_pred.py > gpurun_out/ncu_pred.log 2>&1
