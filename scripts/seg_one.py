"""One segmented launch (after one warm-up) of config 4 or a single config, for ncu:
    python scripts/seg_one.py {config4|config1|config3} [W]"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

name = sys.argv[1]
if len(sys.argv) > 2:
    os.environ["TWB_SIM_SEG_W"] = sys.argv[2]
sw = presets.sweep_1024() if name == "config4" else getattr(presets, name)()
d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
d.run()
d.run()
torch.cuda.synchronize()
