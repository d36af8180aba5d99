"""Iteration mix of the event loop over config 5 (TWB_PROFILE_PHASES build, stride 32):
how many loop iterations are macro runs, single steps (K = 1), admissions, idle jumps,
with > 32 active requests, and the cycle shares of the phases."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_65536() if sys.argv[1:] != ["1024"] else presets.sweep_1024()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
prof = torch.zeros(32 * len(sw), dtype=torch.int64, device="cuda")
_lib.load().tw_sim_set_profile(prof.data_ptr())
dev.run()
torch.cuda.synchronize()
_lib.load().tw_sim_set_profile(None)
pr = prof.view(-1, 32).cpu().numpy().astype(np.float64)
res = dev.fetch().results
cyc = pr[:, 0]
it = pr[:, 1] + pr[:, 2]
names = {1: "normal(K=1)", 2: "runs", 3: "run_steps", 4: "tk_cyc", 7: "arr_cyc", 8: "plan_cyc", 9: "adm_cyc",
         10: "pred_cyc", 11: "apply_cyc", 12: "pred_misses", 13: "tk_calls", 14: "tk_fast", 15: "tk_loops",
         16: "walk_cyc", 17: "fast_cyc", 18: "miss_cyc", 19: "it_adm", 20: "it_wait", 21: "it_wide", 22: "body_cyc",
         23: "it_chunk", 24: "it_k1", 25: "it_idle", 26: "idle_cyc"}
print(f"configs {len(sw)}; iterations per config mean {it.mean():.0f}; steps per config {res['steps'].mean():.0f}")
for k, nm in names.items():
    v = pr[:, k]
    if nm.endswith("cyc"):
        print(f"{nm:12s} {100 * v.sum() / cyc.sum():5.1f}% of cycles")
    else:
        print(f"{nm:12s} {v.sum() / it.sum():7.3f} per iteration ({v.mean():9.1f} per config)")
for model, sel in (("8b", sw.cfgs["pred_id"] < 8), ("70b", sw.cfgs["pred_id"] >= 8)):
    print(model, f"iters {it[sel].mean():.0f}, K=1 {pr[sel, 1].sum() / it[sel].sum():.2f}, adm {pr[sel, 19].sum() / it[sel].sum():.2f}, "
          f"idle/config {pr[sel, 25].mean():.0f}, wide {pr[sel, 21].sum() / it[sel].sum():.3f}, cyc/iter {cyc[sel].sum() / it[sel].sum():.0f}")
