"""Time k_predict_features (2^27 random queries over the 16 calibration tables)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

r = bench.predictor_roofline(torch.device("cuda", 0), 6539.9)
print(json.dumps({k: r[k] for k in ("achieved", "frac", "ms_per_launch", "predictions_per_s")}))
