"""The heaviest config of config 5 alone: serial loop vs segments, with segment statistics."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

full = presets.sweep_65536()
c = int(sys.argv[1]) if len(sys.argv) > 1 else 64315
sw = full.subset([c])
print(sw.configs[0].label)
for env in ({"TWB_SIM_SEG": "0"}, {}, {"TWB_SIM_SEG_W": "16"}, {"TWB_SIM_SEG_W": "32"}, {"TWB_SIM_SEG_W": "128"}):
    for k in ("TWB_SIM_SEG", "TWB_SIM_SEG_W"):
        os.environ.pop(k, None)
    os.environ.update(env)
    d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    _lib.load().tw_sim_set_seg_stats(st.data_ptr())
    d.run()
    torch.cuda.synchronize()
    _lib.load().tw_sim_set_seg_stats(None)
    ms = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); d.run(); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
    r = d.fetch().results[0]
    print(env, f"{min(ms):.3f} ms", "steps", int(r["steps"]), "stats", st.cpu().numpy().tolist())
