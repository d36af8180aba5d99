"""Config 5 sweep time under a given library build, tolerating older ABIs (entry points the
build lacks are stubbed): python scripts/ab_c5_lib.py LIB [reps]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402

path = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
raw = ctypes.CDLL(path)
for name in list(_lib._SIGNATURES):
    if not hasattr(raw, name):
        del _lib._SIGNATURES[name]
lib = _lib.load(path)
if not hasattr(raw, "tw_sim_seg_scratch_bytes"):
    lib.tw_sim_seg_scratch_bytes = lambda n, r: 0
from paper_2601_00397_b200.sweep import DeviceSweep, estimate_cost  # noqa: E402

sw = presets.sweep_65536()
order = np.argsort(-estimate_cost(sw.pset, sw.cfgs, sw.workloads), kind="stable").astype(np.int32)
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
print(f"{path}: " + " ".join(f"{x:.2f}" for x in ms), flush=True)
