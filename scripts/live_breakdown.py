"""Where a resident-service predict goes: ctypes call with an empty batch (round trip only)
vs a 6-slot batch vs the Python predict_one wrapper."""
import ctypes
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_00397_b200 import _lib, presets  # noqa: E402
from paper_2601_00397_b200.predictor import BatchComposition, DecodeSlot, PrefillChunk  # noqa: E402

pred = presets.calibration_set().predictors[0]
batch = BatchComposition(prefill_chunks=(PrefillChunk("p", 384, 0),),
                         decodes=tuple(DecodeSlot(f"d{i}", 500 + i) for i in range(5)))
sv = pred.predictor_set.service()
fn = _lib.load().tw_service_predict
out = ctypes.c_int64()
ref = ctypes.byref(out)
buf = np.array([384, -1, -1, -1, -1, -1, 0, 500, 501, 502, 503, 504], np.int32)
res = {}
for name, n in (("empty", 0), ("six_slots", 6)):
    for _ in range(200):
        fn(sv._h, buf.ctypes.data, n, 0, ref)
    t = time.perf_counter()
    for _ in range(5000):
        fn(sv._h, buf.ctypes.data, n, 0, ref)
    res[name + "_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
t = time.perf_counter()
for _ in range(5000):
    sv.predict_one(batch)
res["predict_one_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
t = time.perf_counter()
for _ in range(5000):
    sv.predict_slots(batch)
res["predict_slots_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
ffn = _lib.load().tw_service_predict_features
for _ in range(200):
    ffn(sv._h, 384, 5, 2510, 0, ref)
t = time.perf_counter()
for _ in range(5000):
    ffn(sv._h, 384, 5, 2510, 0, ref)
res["features_call_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
assert sv.predict_one(batch) == sv.predict_slots(batch)
t = time.perf_counter()
for _ in range(5000):
    fn  # noqa: B018
    _ = (batch.total_prefill_tokens, batch.num_decodes)
res["python_features_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
sys.path.insert(0, "baseline/_ref")
try:
    from timewarp.predictor import TablePredictor as RefTP  # the reference, for scale
    from paper_2601_00397_b200 import calibration
    rp = RefTP.from_csv(calibration.csv_path("8b", 1, 1), allow_extrapolation=True)
    from timewarp.predictor import BatchComposition as RB, DecodeSlot as RD, PrefillChunk as RC
    rbatch = RB(prefill_chunks=(RC("p", 384, 0),), decodes=tuple(RD(f"d{i}", 500 + i) for i in range(5)))
    t = time.perf_counter()
    for _ in range(5000):
        rp.predict(rbatch)
    res["reference_python_predict_us"] = round((time.perf_counter() - t) / 5000 * 1e6, 2)
except Exception as exc:  # noqa: BLE001
    res["reference_error"] = repr(exc)
sv.close()
print(json.dumps(res))
