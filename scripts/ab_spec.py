"""A/B: config 5 restricted to one class (PP=2, prefill-prioritized), generic loop vs a build
specialised for that class (TWB_SPEC_S / TWB_SPEC_POL): python scripts/ab_spec.py LIB"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402

lib = _lib.load(sys.argv[1])
from paper_2601_00397_b200.sweep import DeviceSweep, estimate_cost  # noqa: E402

full = presets.sweep_65536()
sel = np.flatnonzero((full.cfgs["pp_stages"] == 2) & (full.cfgs["policy"] == 1))
sw = full.subset(sel)
order = np.argsort(-estimate_cost(sw.pset, sw.cfgs, sw.workloads), kind="stable").astype(np.int32)
d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True, order=order)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
d.run()
torch.cuda.synchronize()
ms = []
for _ in range(5):
    flush.fill_(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); d.run(); e.record(); e.synchronize()
    ms.append(s.elapsed_time(e))
r = d.fetch().results
print(f"{sys.argv[1]}: {len(sw)} configs, " + " ".join(f"{x:.2f}" for x in ms), "digest-sum", int(r["digest"].astype(np.uint64).sum()) & 0xffffffff)
