mkdir -p gpurun_out
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_pmb4.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_predict_features -s 2 -c 1 -o gpurun_out/prof_pred_f64 python scripts/ab_pred.py > gpurun_out/ncu_pred.log 2>&1
