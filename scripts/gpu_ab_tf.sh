mkdir -p gpurun_out; rm -f gpurun_out/ab_tf.log
for r in 1 2; do for lib in t0 tf1 tf2 tf12; do
  TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_$lib.so timeout 300 python scripts/ab_c5.py model 3 >> gpurun_out/ab_tf.log 2>&1
done; done
cat gpurun_out/ab_tf.log
