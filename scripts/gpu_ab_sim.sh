# parity of the combined k_sim variant, then A/B of every variant (1,024 and 65,536 configs), then the live-engine drop-in test
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_${AB_CHECK:-all}.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sim or sweep" > gpurun_out/pytest_ab.log 2>&1
rm -f gpurun_out/ab.log; bash scripts/ab.sh
AB_VARIANTS="${AB65_VARIANTS:-base all}" bash scripts/ab_65k.sh
timeout 900 python -m pytest tests/test_live_engine.py -x -q > gpurun_out/pytest_live.log 2>&1
tail -3 gpurun_out/pytest_ab.log gpurun_out/pytest_live.log; cat gpurun_out/ab.log gpurun_out/ab_65k.log
