"""Time the fused extraction kernel (bench.extraction_roofline) for A/B runs."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

r = bench.extraction_roofline(torch.device("cuda", 0), 6449.1)
print(json.dumps({k: r[k] for k in ("achieved", "frac", "ms_per_launch", "batches_per_s", "bytes_per_batch")}))
