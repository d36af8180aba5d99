mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py -x -q > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 600 python scripts/ab_seg.py 0 4 8 16 32 > gpurun_out/ab_seg.log 2>&1
tail -n 30 gpurun_out/pytest_seg.log; cat gpurun_out/ab_seg.log
