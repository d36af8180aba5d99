"""Busy-period segments A/B: ms per launch of config 4 (1,024 configs) and configs 1-3,
serial loop (TWB_SIM_SEG=0) vs segmented with several segment counts (TWB_SIM_SEG_W).
    python scripts/ab_seg.py [W ...]"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(sw, env, reps=5):
    os.environ.pop("TWB_SIM_SEG", None)
    os.environ.pop("TWB_SIM_SEG_W", None)
    os.environ.update(env)
    d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
    d.run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); d.run(); e.record(); e.synchronize()
        ms.append(s.elapsed_time(e))
    res = d.fetch().results
    del d
    return sorted(ms)[len(ms) // 2], res


ws = [int(x) for x in sys.argv[1:]] or [0]
for name, sw in (("config4", presets.sweep_1024()), ("config1", presets.config1()), ("config2", presets.config2()),
                 ("config3", presets.config3())):
    base, r0 = timed(sw, {"TWB_SIM_SEG": "0"})
    line = [f"{name}: serial {base:.3f} ms"]
    for w in ws:
        env = {"TWB_SIM_SEG_W": str(w)} if w else {}
        ms, r = timed(sw, env)
        same = all((r[f] == r0[f]).all() for f in r0.dtype.names)
        line.append(f"W={w or 'auto'} {ms:.3f} ms ({'same' if same else 'DIFFERENT'})")
    print("; ".join(line), flush=True)
