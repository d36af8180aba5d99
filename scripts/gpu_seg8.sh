mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py -x -q > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"k_seg_tk|k_sim_seg" python scripts/seg_one.py config4 > gpurun_out/segtk.csv 2>&1
timeout 300 python scripts/ab_env.py > gpurun_out/ab_tk.log 2>&1
tail -n 2 gpurun_out/pytest_seg.log; cat gpurun_out/ab_tk.log; grep -h "gpu__time_duration\|inst_executed" gpurun_out/segtk.csv | cut -d, -f5,13,15 | tail -4
