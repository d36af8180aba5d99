# metrics: this build vs the one without the exact-sum guard (libtwb200_base.so), alternating
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "metrics or summary" 2>&1 | tail -1
for r in 1 2 3; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_base.so timeout 300 python scripts/ab_metrics2.py 65536 | cut -c1-60 | sed 's/^/[base] /'
  timeout 300 python scripts/ab_metrics2.py 65536 | cut -c1-60 | sed 's/^/[new] /'
done
