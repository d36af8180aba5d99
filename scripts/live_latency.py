"""Single-batch predict() latency (the live engine's per-step call, engine.py:684)."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2601_00397_b200 import presets  # noqa: E402
from paper_2601_00397_b200.predictor import BatchComposition, DecodeSlot, PrefillChunk  # noqa: E402

pred = presets.calibration_set().predictors[0]
batch = BatchComposition(prefill_chunks=(PrefillChunk("p", 384, 0),),
                         decodes=tuple(DecodeSlot(f"d{i}", 500 + i) for i in range(5)))
for _ in range(200):
    pred.predict(batch)
res = {}
for name, fn in (("predict_launch_sync", lambda: pred.predict(batch)),
                 ("csr_path", lambda: pred.predictor_set.predict_batches([batch], [0]))):
    t = time.perf_counter()
    for _ in range(2000):
        fn()
    res[name + "_us"] = round((time.perf_counter() - t) / 2000 * 1e6, 2)
res["value_ns"] = pred.predict(batch)
sv = pred.predictor_set.service()  # resident service: nothing may synchronise the device while it runs
t = time.perf_counter()
for _ in range(2000):
    sv.predict_one(batch)
res["resident_service_us"] = round((time.perf_counter() - t) / 2000 * 1e6, 2)
t = time.perf_counter()
for _ in range(2000):
    sv.predict_slots(batch)
res["resident_service_slots_us"] = round((time.perf_counter() - t) / 2000 * 1e6, 2)
sys.path.insert(0, "baseline/_ref")
try:  # the reference's own predict() on the same batch, for scale
    from timewarp.predictor import BatchComposition as RB, DecodeSlot as RD, PrefillChunk as RC
    from timewarp.predictor import TablePredictor as RT

    from paper_2601_00397_b200 import calibration
    rp = RT.from_csv(calibration.csv_path("8b", 1, 1), allow_extrapolation=True)
    rbatch = RB(prefill_chunks=(RC("p", 384, 0),), decodes=tuple(RD(f"d{i}", 500 + i) for i in range(5)))
    assert rp.predict(rbatch) == res["value_ns"]
    t = time.perf_counter()
    for _ in range(2000):
        rp.predict(rbatch)
    res["reference_python_predict_us"] = round((time.perf_counter() - t) / 2000 * 1e6, 2)
except ImportError:
    pass
assert sv.predict_one(batch) == res["value_ns"] == int(pred.predictor_set.predict_batches([batch], [0])[0])
sv.close()
print(json.dumps(res))
