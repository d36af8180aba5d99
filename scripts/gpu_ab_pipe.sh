for r in 1 2; do
for v in "" pipe pipe768 t768; do
  if [ -n "$v" ]; then L="TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$v.so"; else L=""; fi
  echo -n "[$v] "; env $L timeout 300 python scripts/ab_pred.py 2>&1 | tail -1
done; done
