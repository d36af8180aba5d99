"""End-to-end step (HostSweep) of config 5 (or config 4 with `1024`): the streamed copy-back
(default above 256 MB of outputs) vs one copy after the kernel (chunk = every config), and
the kernel alone for reference."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import HostSweep  # noqa: E402

sw = presets.sweep_65536() if len(sys.argv) < 2 else presets.sweep_1024()
out = {}
for mode in ("streamed", "copy_after", "streamed", "copy_after"):
    host = HostSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True, zero_copy=False)
    if mode == "copy_after":
        host.STREAM_CHUNK_CONFIGS = 1 << 30
    for _ in range(2):
        host.run_from_host()
    torch.cuda.synchronize()
    for what, fn in ((mode, host.run_from_host), ("kernel_only", host.run)):
        ms = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize()
            ms.append(a.elapsed_time(b))
        out.setdefault(what, []).append(round(float(np.median(ms)), 2))
    del host
    torch.cuda.empty_cache()
print(json.dumps(out))
