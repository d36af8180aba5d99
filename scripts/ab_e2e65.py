"""Config-5 end-to-end step (HostSweep) with zero-copy outputs vs a copy-back after the kernel."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import HostSweep  # noqa: E402

sw = presets.sweep_65536() if len(sys.argv) < 2 else presets.sweep_1024()
out = {}
for zc in (True, False, True, False):
    host = HostSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True, zero_copy=zc)
    for _ in range(2):
        host.run_from_host()
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); host.run_from_host(); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
    out.setdefault(f"zero_copy={zc}", []).append(round(float(np.median(ms)), 2))
    del host
    torch.cuda.empty_cache()
print(json.dumps(out))
