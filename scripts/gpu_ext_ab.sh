# extraction kernel: parity tests, then per-warp (product) vs producer-warp A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "extraction or live_single" > gpurun_out/pytest_ext.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ext.log
AB_VARIANTS="t8 t6 t4 prod" bash scripts/ab_ext2.sh
tail -3 gpurun_out/pytest_ext.log
