mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "65536 or throughput or blob_larger or slot or invariant or host_sweep" > gpurun_out/pytest_cls.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cls.log
for r in 1 2; do
  TWB_SIM_CLS=0 timeout 300 python scripts/ab_c5.py model 3 | sed 's/^/[generic] /'
  timeout 300 python scripts/ab_c5.py model 3 | sed 's/^/[classes] /'
done > gpurun_out/ab_cls.log 2>&1
tail -n 2 gpurun_out/pytest_cls.log; cat gpurun_out/ab_cls.log
