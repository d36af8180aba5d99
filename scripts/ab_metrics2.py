"""tw_metrics_many with the TPOT rows in scratch (k_metrics_tpot) vs without (one thread per
config sums in k_metrics): python scripts/ab_metrics2.py [1024|65536]"""
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_65536() if sys.argv[1:] == ["65536"] else presets.sweep_1024()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
dev.run()
dev.run_metrics()
full = dev.d_met_scratch
out = {}
for name, scr in (("tpot_kernel", full), ("in_kernel_sum", None)):
    dev.d_met_scratch = scr
    for _ in range(3):
        dev.run_metrics()
    torch.cuda.synchronize()
    d = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dev.run_metrics(); b.record(); b.synchronize()
        d.append(a.elapsed_time(b))
    m = dev.fetch_metrics()
    out[name] = {"ms": round(statistics.median(d), 4), "ok": bool((m["status"] == 0).all()),
                 "tpot_mean_bits": int(np.asarray(m["tpot"]["mean"]).view(np.int64).sum())}
print(json.dumps(out))
