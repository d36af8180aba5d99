mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "predict or extraction or csr or known_answers or larger_than" 2>&1 | tail -3
AB_VARIANTS="old new" timeout 900 bash scripts/ab_both.sh; cat gpurun_out/ab_both.log
