"""Time the bulk Timekeeper min-advance (bench.timekeeper_roofline) for A/B runs."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

print(json.dumps(bench.timekeeper_roofline(torch.device("cuda", 0), 6449.1)))
