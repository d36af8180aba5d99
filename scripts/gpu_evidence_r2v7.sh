# round-2 v7 evidence (session 4): tests, smoke, bench, reference arm, 1-rank NCCL run, launch
# list, and ncu --set full of the kernels changed this session (k_metrics, k_sim_join)
mkdir -p gpurun_out
nproc > gpurun_out/box.txt; nvidia-smi -L >> gpurun_out/box.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29501 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-projection --no-config4 --no-configs13 > gpurun_out/bench_nccl1.log 2>&1; echo "nccl1 rc=$?" >> gpurun_out/bench_nccl1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-projection --no-configs13 > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_sim_join|k_seg_plan" -s 2 -c 2 -f -o gpurun_out/prof_segjoin python scripts/seg_one.py config4 > gpurun_out/ncu_segjoin.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_metrics -s 2 -c 2 -f -o gpurun_out/prof_metrics python scripts/ab_metrics.py 65536 > gpurun_out/ncu_metrics.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 400 gpurun_out/bench.log; tail -c 300 gpurun_out/bench_ref.log
