"""Quantify the in-loop Timekeeper model against the reference's live stack under PP.

The device event loop drives each config's BarrierCore with parked workers EXEMPT
("idealized"). The reference's live WorkerGrid leaves a finished stage's
workers idle in commands.get(), registered and non-exempt (engine.py:394-415), so later
stages' rounds cannot resolve and advance at wall pace (client.py:193-214 waits out the
remaining distance). This script runs the UNMODIFIED reference live stack (baseline/_ref,
runner.run_benchmark in timewarp mode: engine subprocess + TCP Timekeeper, real clock)
for TP x PP grids and compares its measured wall time and broadcast count with the
model's (seq, FakeClock wall) from the C oracle on the same arrivals, table and engine.
Writes profiles/r02_tk_live_vs_model.json. The event timelines are identical either way
(checked here too)."""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = os.path.join(ROOT, "baseline", "_ref")

RUN = r'''
import json, sys
from timewarp.runner import run_benchmark
doc = json.loads(sys.argv[1]); out = sys.argv[2]
rep = run_benchmark(doc, "timewarp", out, verify_log=False)
seq = 0
with open(out + "/timekeeper_log.jsonl") as fh:
    for line in fh:
        r = json.loads(line)
        if r.get("event") == "broadcast":
            seq = max(seq, int(r["seq"]))
ev = [json.loads(l) for l in open(out + "/engine_events.jsonl") if l.strip()]
print(json.dumps({"virtual_ns": rep.virtual_elapsed_ns, "wall_ns": rep.wall_elapsed_ns, "seq": seq,
                  "epoch_ns": rep.epoch_ns, "events": [[e["request_id"], e["kind"], int(e["virtual_ts_ns"]) - rep.epoch_ns, e["step"]] for e in ev]}))
'''


def model(doc, tp, pp):
    from oracle import oracle as orc
    from paper_2601_00397_b200 import calibration
    from paper_2601_00397_b200.predictor import PredictorSet, TablePredictor
    from paper_2601_00397_b200.sweep import EngineConfig, SchedulingPolicy, SweepConfig, config_array
    from paper_2601_00397_b200.workload import WorkloadSpec, pack_arrays, poisson_arrays

    wl = pack_arrays([poisson_arrays(WorkloadSpec.from_doc(doc["workload"]))])
    e = doc["engine"]
    eng = EngineConfig(chunk_size=e["chunk_size"], max_batch_tokens=e["max_batch_tokens"], max_running=e["max_running"],
                       kv_block_tokens=e["kv_block_tokens"], kv_capacity_blocks=e["kv_capacity_blocks"],
                       policy=SchedulingPolicy(e["policy"]), workers_per_replica=tp, pp_stages=pp)
    pset = PredictorSet([TablePredictor.from_csv(calibration.csv_path("8b", tp, pp), allow_extrapolation=True)])
    cfgs = config_array([SweepConfig(engine=eng, pred_id=0, workload_id=0, timekeeper=True,
                                     tk_cooldown_ns=doc["timekeeper"]["jitter_cooldown_us"] * 1000)])
    res, ev, *_ = orc.sim_many(pset.blob, cfgs, wl.wl_off, wl.offset_ns, wl.prompt, wl.output)
    r = res[0]
    return {"virtual_ns": int(r["final_now_ns"]), "fake_wall_ns": int(r["tk_wall_ns"]), "seq": int(r["tk_seq"]),
            "steps": int(r["steps"]), "digest": int(np.uint64(r["digest"]))}


def main():
    from oracle.oracle import digest_of_docs

    cases = [(2, 1), (2, 2), (4, 2)]
    out = {"note": __doc__.split("\n\n")[1].replace("\n", " "), "cases": []}
    for tp, pp in cases:
        doc = {"workload": {"source": "poisson", "qps": 16, "seed": 3, "num_requests": 24,
                            "prompt_tokens": {"kind": "uniform", "low": 64, "high": 1024},
                            "output_tokens": {"kind": "uniform", "low": 4, "high": 32}},
               "engine": {"chunk_size": 256, "max_batch_tokens": 1024, "max_running": 16, "kv_block_tokens": 16,
                          "kv_capacity_blocks": 2048, "policy": "mixed", "workers_per_replica": tp, "pp_stages": pp},
               "predictor": {"kind": "table", "path": __import__("paper_2601_00397_b200.calibration",
                                                                 fromlist=["x"]).csv_path("8b", tp, pp),
                             "allow_extrapolation": True},
               "timekeeper": {"jitter_cooldown_us": 500}}
        with tempfile.TemporaryDirectory() as td:
            env = dict(os.environ, PYTHONPATH=REF)
            p = subprocess.run([sys.executable, "-c", RUN, json.dumps(doc), td], env=env, capture_output=True,
                               text=True, timeout=1800)
            if p.returncode != 0:
                raise SystemExit(p.stderr[-3000:])
            live = json.loads(p.stdout.strip().splitlines()[-1])
        m = model(doc, tp, pp)
        evs = [{"request_id": a, "kind": b, "virtual_ts_ns": c, "step": d} for a, b, c, d in live["events"]]
        order = sorted({e["request_id"] for e in evs})
        idx = {rid: k for k, rid in enumerate(sorted(order, key=lambda s: int(s[1:]) if s[1:].isdigit() else s))}
        rec = {"tp": tp, "pp": pp, "actors": 1 + tp * pp,
               "live": {"virtual_s": live["virtual_ns"] / 1e9, "wall_s": live["wall_ns"] / 1e9, "seq": live["seq"],
                        "speedup": live["virtual_ns"] / max(live["wall_ns"], 1)},
               "model_idealized": {"virtual_s": m["virtual_ns"] / 1e9, "fake_wall_s": m["fake_wall_ns"] / 1e9,
                                   "seq": m["seq"], "speedup": m["virtual_ns"] / max(m["fake_wall_ns"], 1)},
               "same_virtual_span": live["virtual_ns"] == m["virtual_ns"],
               "same_events_digest": digest_of_docs(evs, idx) == m["digest"]}
        rec["wall_ratio_live_over_model"] = rec["live"]["wall_s"] / max(rec["model_idealized"]["fake_wall_s"], 1e-9)
        out["cases"].append(rec)
        print(json.dumps(rec), flush=True)
    with open(os.path.join(ROOT, "profiles", "r02_tk_live_vs_model.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
