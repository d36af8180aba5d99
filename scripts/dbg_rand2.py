"""Debug: random sweep vs the C oracle, the configs that differ."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_segments as T  # noqa: E402
from oracle import oracle as orc  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
pset, wl, ca, _ = T._random_sweep(seed)
out, _ = T._run(pset, wl, ca, {"TWB_SIM_SEG": "0"})
res, _, first, finish = orc.sim_many(pset.blob, ca, wl.wl_off, wl.offset_ns, wl.prompt, wl.output, per_request=True)
bad = [c for c in range(len(ca)) if any(out.results[f][c] != res[f][c] for f in T.FIELDS)]
print("bad", len(bad), bad[:10])
for c in bad[:5]:
    cf = ca[c]
    print(c, {k: int(cf[k]) for k in ("chunk_size", "max_batch_tokens", "max_running", "kv_block_tokens", "kv_capacity_blocks",
                                      "pp_stages", "workers_per_replica", "policy", "pred_id", "workload_id", "tk_cooldown_ns",
                                      "flags", "epoch_ns")}, "n", int(wl.wl_off[cf["workload_id"] + 1] - wl.wl_off[cf["workload_id"]]))
    for f in T.FIELDS:
        if out.results[f][c] != res[f][c]:
            print("    ", f, "gpu", int(out.results[f][c]), "oracle", int(res[f][c]))
