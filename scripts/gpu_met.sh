timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "metrics" 2>&1 | tail -2
timeout 300 python scripts/ab_metrics2.py 1024
timeout 300 python scripts/ab_metrics2.py 65536
