# parity of variant $AB_CHECK (sim tests) then A/B of $AB_VARIANTS at 1,024 and 65,536 configs
mkdir -p gpurun_out
TWB200_ALLOW_LIB_OVERRIDE=1 TWB200_LIB=paper_2601_00397_b200/lib/libtwb200_${AB_CHECK}.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sim or sweep" > gpurun_out/pytest_ab.log 2>&1
tail -1 gpurun_out/pytest_ab.log
bash scripts/ab_occ.sh
