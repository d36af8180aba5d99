"""Debug: where the segmented run's stamps differ from the serial loop's (stop-early configs)."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_segments import _run  # noqa: E402

from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.predictor import LinearPredictor, PredictorSet  # noqa: E402

sw = presets.config1()
cfgs = np.repeat(sw.cfgs, 6)
cfgs["kv_capacity_blocks"][0] = 100
cfgs["kv_capacity_blocks"][1] = 126
cfgs["max_batch_tokens"][2:4] = 4096
cfgs["chunk_size"][2:4] = 4096
pset = PredictorSet([sw.pset.predictors[cfgs["pred_id"][0]], LinearPredictor(10000.0, -4.9, 30.0),
                     LinearPredictor(9000.0, -4.0, 20.0)])
cfgs["pred_id"][:] = 0
cfgs["pred_id"][2] = 1
cfgs["pred_id"][3] = 2
cfgs["max_running"][4] = 1
ser, _ = _run(pset, sw.workloads, cfgs, {"TWB_SIM_SEG": "0"})
seg, _ = _run(pset, sw.workloads, cfgs, {})
for c in range(6):
    lo, hi = ser.req_base[c], ser.req_base[c + 1]
    a, b = ser.first_ns[lo:hi], seg.first_ns[lo:hi]
    f, g = ser.finish_ns[lo:hi], seg.finish_ns[lo:hi]
    df = np.flatnonzero(a != b)
    dg = np.flatnonzero(f != g)
    r = ser.results[c]
    print(c, "status", r["status"], seg.results[c]["status"], "steps", r["steps"], "first diffs", len(df), df[:12],
          "finish diffs", len(dg), dg[:12])
    if len(df):
        print("   ser first", a[df[:6]], "seg", b[df[:6]])
    if len(dg):
        print("   ser fin", f[dg[:6]], "seg", g[dg[:6]])
    print("   last stamped (ser)", np.flatnonzero(a >= 0).max() if (a >= 0).any() else -1,
          "unset first count ser/seg", (a < 0).sum(), (b < 0).sum())
