"""Time one tw_sim_many launch over BASELINE config 5 (65,536 configs) on one GPU (A/B helper)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_65536()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
import os  # noqa: E402

if os.environ.get("STAGE") == "core":  # A/B against builds that stage the blob at every size
    dev.stage_bytes = sw.pset.core_nbytes
dev.run()
torch.cuda.synchronize()
ms = []
for _ in range(2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dev.run(); e.record(); e.synchronize()
    ms.append(s.elapsed_time(e))
r = dev.fetch().results
print(json.dumps({"ms": [round(m, 2) for m in ms], "ok": bool((r["status"] == 0).all()),
                  "steps": int(r["steps"].sum()), "launch": _lib.last_sim_launch()}))
