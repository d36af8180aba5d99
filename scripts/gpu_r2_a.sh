# round 2: GPU parity after digest v2, the new bench line, 1-rank NCCL and 2-rank gloo dry runs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29501 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-projection --no-config4 > gpurun_out/bench_nccl1.log 2>&1; echo "nccl1 rc=$?" >> gpurun_out/bench_nccl1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 3 --warmup 3 --share-device > gpurun_out/bench_dry2.log 2>&1; echo "dry2 rc=$?" >> gpurun_out/bench_dry2.log
tail -2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench.log; tail -c 300 gpurun_out/bench_nccl1.log gpurun_out/bench_dry2.log
