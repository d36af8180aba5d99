for r in 1 2; do
for v in "" bpt2 bpt4; do
  if [ -n "$v" ]; then L="TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so"; else L=""; fi
  echo -n "[$v] "; env $L timeout 300 python scripts/ab_ext.py 2>&1 | tail -1
done; done
for v in bpt2 bpt4; do env TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "extraction" 2>&1 | tail -1; done
