mkdir -p gpurun_out
python scripts/prof_one.py 24 > gpurun_out/prof_one.log 2>&1
python scripts/prof_one.py 273 >> gpurun_out/prof_one.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sim -s 1 -c 1 -o gpurun_out/prof_one python scripts/prof_one.py 24 > gpurun_out/ncu_one.log 2>&1
