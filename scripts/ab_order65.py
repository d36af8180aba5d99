"""ab_order.py at BASELINE config 5 (65,536 configs, throughput variant)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402
from paper_2601_00397_b200._device import to_device  # noqa: E402

sw = presets.sweep_65536()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
prof = torch.zeros(16 * len(sw), dtype=torch.int64, device="cuda")
_lib.load().tw_sim_set_profile(prof.data_ptr())
dev.run()
torch.cuda.synchronize()
_lib.load().tw_sim_set_profile(None)
cyc = prof.view(-1, 16)[:, 0].cpu().numpy()


def timed(order):
    dev.order = np.ascontiguousarray(order, np.int32)
    dev.d_order = to_device(dev.order, dev.device)
    for _ in range(2):
        dev.run()
    ms = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dev.run(); e.record(); e.synchronize()
        ms.append(s.elapsed_time(e))
    return round(float(np.median(ms)), 3)


est = dev.order.copy()
rank_est = np.empty(len(est), int); rank_est[est] = np.arange(len(est))
out = {"estimate": timed(est), "measured": timed(np.argsort(-cyc, kind="stable")),
       "reverse_measured": timed(np.argsort(cyc, kind="stable")), "identity": timed(np.arange(len(cyc))),
       "corr_est_vs_cycles": float(np.corrcoef(-rank_est, cyc)[0, 1]),
       "cyc_ms_max_median": [round(cyc.max() / 1.965e6, 3), round(float(np.median(cyc)) / 1.965e6, 3)]}
print(json.dumps(out))
