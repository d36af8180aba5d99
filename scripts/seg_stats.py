"""Segmented-path statistics (tw_sim_set_seg_stats) and ms per launch for config 4 and
configs 1-3 at several segment counts:  python scripts/seg_stats.py [W ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

ws = [int(x) for x in sys.argv[1:]] or [0]
for name in ("config4", "config1", "config3"):
    sw = presets.sweep_1024() if name == "config4" else getattr(presets, name)()
    for w in ws:
        if w:
            os.environ["TWB_SIM_SEG_W"] = str(w)
        else:
            os.environ.pop("TWB_SIM_SEG_W", None)
        d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
        st = torch.zeros(8 * len(sw), dtype=torch.int32, device="cuda")
        _lib.load().tw_sim_set_seg_stats(st.data_ptr())
        d.run()
        torch.cuda.synchronize()
        _lib.load().tw_sim_set_seg_stats(None)
        s = st.view(-1, 8).cpu().numpy().astype(np.int64)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); d.run(); e1.record(); e1.synchronize()
        print(f"{name} W={w or 'auto'}: {e0.elapsed_time(e1):.3f} ms; segments {s[:,0].sum()}, joined {s[:,1].sum()}, "
              f"serial pieces {s[:,2].sum()}, tk refused {s[:,3].sum()}, overflowed {s[:,4].sum()}, "
              f"not converged {s[:,5].sum()}", flush=True)
        del d
