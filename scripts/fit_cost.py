"""Fit the sweep cost model (paper_2601_00397_b200/cost_model.json) to measured per-config
cycles: `gpurun_out/prof65.npz` from scripts/prof_sim65.py (config 5 with tw_sim_set_profile).

log(cycles) ~ linear in the numeric features of sweep.cost_features and their pairwise
products (least squares). Prints the fit quality and the LPT shard imbalance it gives at
N = 2, 4, 8 with the measured cycles as the truth."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.distributed import partition  # noqa: E402
from paper_2601_00397_b200.sweep import COST_MODEL_PATH, cost_design, cost_features  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof65.npz"
full = presets.sweep_65536()
cyc = np.load(src)["cyc"].astype(np.float64)
names, F = cost_features(full.pset, full.cfgs, full.workloads)
X, terms = cost_design(names, F)
y = np.log(cyc)
coef, *_ = np.linalg.lstsq(X, y, rcond=None)
pred = X @ coef
r2 = 1 - ((y - pred) ** 2).sum() / ((y - y.mean()) ** 2).sum()
est = np.exp(pred)
imb = {}
for N in (2, 4, 8):
    sh = partition(est, N)
    s = [cyc[x].sum() for x in sh]
    imb[N] = round(float(max(s) / np.mean(s)), 5)
doc = {"features": names, "terms": terms, "coef": [float(x) for x in coef],
       "fit": {"source": "config 5 (65,536 configs) per-config cycles, tw_sim_set_profile, one B200",
               "r2_log": round(float(r2), 4), "corr": round(float(np.corrcoef(est, cyc)[0, 1]), 4),
               "lpt_cycle_imbalance": imb}}
json.dump(doc, open(COST_MODEL_PATH, "w"), indent=1)
print(json.dumps(doc["fit"]))
