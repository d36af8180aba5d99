"""Time the fused extraction kernel (bench.extraction_roofline) for A/B runs."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

r = bench.extraction_roofline(torch.device("cuda", 0), 6449.1)
po = r["predictions_only"]
print(json.dumps({"feat_frac": r["frac"], "feat_ms": r["ms_per_launch"], "pred_frac": po["frac"],
                  "pred_ms": po["ms_per_launch"], "pred_frac_56B": round(po["frac"] * 56 / po["bytes_per_batch"], 4)}))
