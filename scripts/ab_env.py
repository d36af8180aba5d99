"""ms per launch of config 4 (and config 1 / 3) under environment variants:
    python scripts/ab_env.py "TWB_SIM_SEG_LAT=1" "TWB_SIM_SEG_LAT=1 TWB_SIM_SEG_STAGE=33056" ..."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
variants = [""] + sys.argv[1:]
sweeps = [("config4", presets.sweep_1024()), ("config1", presets.config1()), ("config3", presets.config3())]
for name, sw in sweeps:
    out = []
    for v in variants:
        env = dict(kv.split("=", 1) for kv in v.split())
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        d = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
        d.run()
        torch.cuda.synchronize()
        ms = []
        for _ in range(7):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); d.run(); b.record(); b.synchronize()
            ms.append(a.elapsed_time(b))
        del d
        for k, x in old.items():
            if x is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = x
        out.append(f"[{v or 'default'}] {sorted(ms)[3]:.3f}")
    print(name, " ".join(out), flush=True)
