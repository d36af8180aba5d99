"""Per-config critical-path profile of k_sim (tw_sim_set_profile) on the 1,024 sweep."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402

sw = presets.sweep_1024()
dev = DeviceSweep(sw.pset, sw.workloads, sw.cfgs, per_request=True)
import os  # noqa: E402
STRIDE = int(os.environ.get("TWB_PROF_STRIDE", "16"))  # 32 for TWB_PROFILE_PHASES builds
prof = torch.zeros(STRIDE * len(sw), dtype=torch.int64, device="cuda")
_lib.load().tw_sim_set_profile(prof.data_ptr())
for _ in range(3):
    dev.run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); dev.run(); e.record(); e.synchronize()
ms = s.elapsed_time(e)
_lib.load().tw_sim_set_profile(None)
pr = prof.view(-1, STRIDE).cpu().numpy()
res = dev.fetch().results
cyc, normal, runs, run_steps, tkc, evc, rounds, arc, plc, adc, prc, apc, misses, tcalls, tfast, tloops = pr.T[:16]
order = np.argsort(-cyc)
print(f"kernel {ms:.2f} ms; max config {cyc.max()/1.965e6:.2f} ms @1.965GHz, median {np.median(cyc)/1.965e6:.2f} ms")
print(f"steps total {res['steps'].sum()}, normal {normal.sum()}, runs {runs.sum()}, run steps {run_steps.sum()}")
print(f"cycles per normal step (approx, all configs) {cyc.sum()/max(1,normal.sum()+runs.sum()):.0f} per normal-or-run")
for c in order[:12]:
    lab = sw.configs[c].label
    print(c, f"{cyc[c]/1.965e6:.2f}ms", "steps", res['steps'][c], "normal", normal[c], "runs", runs[c], "runsteps", run_steps[c],
          f"tk {100*tkc[c]/cyc[c]:.0f}% ev {100*evc[c]/cyc[c]:.0f}% arr {100*arc[c]/cyc[c]:.0f}% plan {100*plc[c]/cyc[c]:.0f}% "
          f"adm {100*adc[c]/cyc[c]:.0f}% pred {100*prc[c]/cyc[c]:.0f}% apply {100*apc[c]/cyc[c]:.0f}% bcasts {rounds[c]} "
          f"pred-misses {misses[c]} tk calls/fast/loop-iters {tcalls[c]}/{tfast[c]}/{tloops[c]}", lab)
# fit cycles ~ a*normal + b*runs + c*run_steps
A = np.stack([normal, runs, run_steps], 1).astype(float)
coef, *_ = np.linalg.lstsq(A, cyc.astype(float), rcond=None)
print("fit cycles/normal step, /run, /run step:", coef.round(1))
if STRIDE == 32:
    names = ["walk_cyc", "fast_cyc", "miss_cyc", "it_adm", "it_wait", "it_wide", "body_cyc", "it_chunk", "it_k1",
             "it_idle", "idle_cyc"]
    for c in order[:3]:
        it = normal[c] + runs[c]
        print(c, "iters", it, {k: int(v) for k, v in zip(names, pr[c, 16:27])},
              f"walk {100*pr[c,16]/cyc[c]:.1f}% fast {100*pr[c,17]/cyc[c]:.1f}% miss {100*pr[c,18]/cyc[c]:.1f}% "
              f"body {100*pr[c,22]/cyc[c]:.1f}% idle {100*pr[c,26]/cyc[c]:.1f}% cyc/iter {cyc[c]/it:.0f}")
json.dump({"ms": ms, "cyc": cyc.tolist(), "normal": normal.tolist(), "runs": runs.tolist(), "run_steps": run_steps.tolist()},
          open("gpurun_out/prof_sim.json", "w"))
