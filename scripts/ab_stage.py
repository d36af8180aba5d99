"""A/B: k_sim staging only the core predictor blob vs the whole blob (bulk-lookup
section for prediction-cache misses) on the 1,024-config sweep."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_1024()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
ref = None
for rep in range(3):
    for name, nbytes in (("core", sw.pset.core_nbytes), ("full", sw.pset.nbytes)):
        dev.stage_bytes = nbytes
        dev.run()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dev.run(); e.record(); e.synchronize()
        r = dev.fetch().results
        if ref is None:
            ref = r.copy()
        assert (r == ref).all()
        print(name, round(s.elapsed_time(e), 3), "ms", flush=True)
