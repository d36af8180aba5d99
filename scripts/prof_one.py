"""Launch k_sim on a single config of the 1,024 sweep (its critical path alone)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 24
sw = presets.sweep_1024().subset([cid])
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
dev.run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); dev.run(); e.record(); e.synchronize()
print(f"config {cid} alone: {s.elapsed_time(e):.3f} ms", sw.configs[0].label)
