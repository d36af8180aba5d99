# A/B the join prefetch: parity of the new lib, then alternating timings vs the HEAD build
timeout 600 python -m pytest tests/test_gpu_segments.py -q -x 2>&1 | tail -1
for r in 1 2; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_base.so timeout 300 python scripts/ab_env.py | sed 's/^/[base] /'
  timeout 300 python scripts/ab_env.py | sed 's/^/[new] /'
done
