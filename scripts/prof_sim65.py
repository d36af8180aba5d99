"""Config 5 (65,536 configs) per-config cycles (tw_sim_set_profile) for the cost-model fit,
plus each LPT shard of N = 2, 4, 8 timed ALONE on this GPU (what rank r of N runs): the
projected strong-scaling curve, under the current estimate_cost and under measured cycles."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.distributed import partition  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep, estimate_cost  # noqa: E402


def timed(dev, reps=3):
    dev.run()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); dev.run(); e.record(); e.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


full = presets.sweep_65536()
dev = DeviceSweep(full.pset, full.workloads, full.cfgs, per_request=True)
prof = torch.zeros(16 * len(full), dtype=torch.int64, device="cuda")
_lib.load().tw_sim_set_profile(prof.data_ptr())
ms_full = timed(dev, 2)
_lib.load().tw_sim_set_profile(None)
cyc = prof.view(-1, 16)[:, 0].cpu().numpy().astype(np.float64)
res = dev.fetch().results
np.savez("gpurun_out/prof65.npz", cyc=cyc, steps=res["steps"], prof=prof.view(-1, 16).cpu().numpy())
del dev
torch.cuda.empty_cache()
est = estimate_cost(full.pset, full.cfgs, full.workloads)
print(f"full sweep {ms_full:.1f} ms; corr(estimate, cycles) = {np.corrcoef(est, cyc)[0, 1]:.3f}", flush=True)
out = {"full_ms": ms_full}
for name, cost in (("estimate", est), ("measured", cyc)):
    for N in (2, 4, 8):
        shards = partition(cost, N)
        ms = []
        for r in range(N):
            sub = full.subset(shards[r])
            order = np.argsort(-cost[shards[r]], kind="stable").astype(np.int32)
            d = DeviceSweep(sub.pset, sub.workloads, sub.cfgs, per_request=True, order=order)
            ms.append(timed(d))
            del d
        pred = [float(cyc[s].sum()) for s in shards]
        out[f"{name}_N{N}"] = {"shard_ms": ms, "cycles_per_shard": pred}
        print(name, N, "shard ms", [round(x, 1) for x in ms], "max/mean", round(max(ms) / np.mean(ms), 4),
              "ideal", round(ms_full / N, 1), "cycle-sum imbalance", round(max(pred) / np.mean(pred), 4), flush=True)
json.dump(out, open("gpurun_out/prof65_shards.json", "w"))
