# lane-per-segment Timekeeper replay: parity (default and the warp kernel), then timings
timeout 600 python -m pytest tests/test_gpu_segments.py -q -x 2>&1 | tail -1
TWB_SEG_TK_LANES=8 timeout 600 python -m pytest tests/test_gpu_segments.py -q -x 2>&1 | tail -1
for r in 1 2; do
  timeout 300 python scripts/ab_env.py "TWB_SEG_TK_LANES=0" "TWB_SEG_TK_LANES=8" "TWB_SEG_TK_LANES=16" "TWB_SEG_TK_LANES=32"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_seg_tk --csv python scripts/ab_env.py "TWB_SEG_TK_LANES=0" "TWB_SEG_TK_LANES=8" 2>/dev/null | grep -v "^==" | awk -F, '{print $5, $(NF)}' | sort | uniq -c | tail -12
