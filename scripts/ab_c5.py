"""Config 5 sweep time under one library (TWB200_LIB) with a given pull order:
   python scripts/ab_c5.py {old|model|measured} [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.predictor import ConstantPredictor, LinearPredictor  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep, estimate_cost  # noqa: E402


def old_estimate(pset, cfgs, wl):  # round-1 estimate_cost: tokens / sqrt(fastest table step)
    tokens = np.array([float(wl.output[wl.wl_off[w]:wl.wl_off[w + 1]].sum()) + 1.0 for w in range(wl.n_workloads)])
    step_us = np.ones(len(pset.predictors))
    for i, p in enumerate(pset.predictors):
        if isinstance(p, ConstantPredictor):
            step_us[i] = max(p.duration_us, 1)
        elif isinstance(p, LinearPredictor):
            step_us[i] = max(abs(p.base_us) + abs(p.per_decode_us), 1.0)
        else:
            step_us[i] = max(min(p._rows.values()), 1)
    return tokens[cfgs["workload_id"]] / np.sqrt(step_us[np.clip(cfgs["pred_id"], 0, len(step_us) - 1)])


kind = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sw = presets.sweep_1024() if "1k" in kind else presets.sweep_65536()
if kind.startswith("old"):
    cost = old_estimate(sw.pset, sw.cfgs, sw.workloads)
elif kind.startswith("measured"):
    cost = np.load("gpurun_out/prof65.npz")["cyc"]
else:
    cost = estimate_cost(sw.pset, sw.cfgs, sw.workloads)
order = np.argsort(-cost, kind="stable").astype(np.int32)
d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True, order=order)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
d.run()
torch.cuda.synchronize()
ms = []
for _ in range(reps):
    flush.fill_(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); d.run(); e.record(); e.synchronize()
    ms.append(s.elapsed_time(e))
import os  # noqa: E402
print(f"{os.environ.get('TWB200_LIB', 'default')} {kind}: " + " ".join(f"{x:.2f}" for x in ms), flush=True)
