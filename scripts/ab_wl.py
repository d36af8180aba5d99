"""Time bulk workload generation (bench.workload_generation) for A/B runs."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import torch  # noqa: E402

print(json.dumps(bench.workload_generation(torch.device("cuda", 0))))
