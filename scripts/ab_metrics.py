"""Time tw_metrics_many over a sweep's stamps (A/B helper): `python scripts/ab_metrics.py [1024|65536]`."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_65536() if sys.argv[1:] == ["65536"] else presets.sweep_1024()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
dev.run()
for _ in range(3):
    dev.run_metrics()
torch.cuda.synchronize()
d = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dev.run_metrics(); b.record(); b.synchronize()
    d.append(a.elapsed_time(b))
m = dev.fetch_metrics()
print(json.dumps({"ms": round(statistics.median(d), 4), "ok": bool((m["status"] == 0).all()),
                  "chk": float(m["tpot"]["mean"].sum())}))
