"""Live-path drop-in: the reference's own live stack with this
engine's predictor inside it.

The reference's ``EmulatedEngine`` runs in its own subprocess (``timewarp.engine_main``),
paced by the reference's Timekeeper over TCP in timewarp mode
(``runner.run_benchmark``, pkg/src/timewarp/runner.py:182). The only change is
``build_predictor`` (pkg/src/timewarp/predictor.py:245), replaced through a
``sitecustomize`` so the engine's per-step call (engine.py:684) lands in
``paper_2601_00397_b200.predictor`` (tw_predict_one_sync on the GPU). The event stream
must equal the reference oracle's with the reference's CPU predictor, event for event:
the assertions of pkg/tests/test_harness_integration.py:77-84.

Needs the reference package installed under ``baseline/_ref`` (the task's one offline
``pip install --target``; git-ignored, shipped to the GPU box with the snapshot) and a
GPU; skipped otherwise. The native-BarrierCore test (§8f row 3) needs no GPU.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import textwrap

import pytest

from paper_2601_00397_b200 import calibration

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "timewarp")),
                                reason="reference not installed under baseline/_ref")

# engine-process hook: the reference's factory, answered by this engine's predictors
SITECUSTOMIZE = textwrap.dedent('''
    import atexit, json, os, sys
    sys.path.insert(0, os.environ["TWB200_ROOT"])
    import timewarp.predictor as _ref_predictor

    _calls = {"n": 0, "kinds": []}

    class _Counted:
        def __init__(self, inner):
            self.inner = inner
        def predict(self, batch, hw=None):
            _calls["n"] += 1
            return self.inner.predict(batch, hw)

    def build_predictor(config):
        from paper_2601_00397_b200 import predictor as _b200
        _calls["kinds"].append(config.get("kind"))
        return _Counted(_b200.build_predictor(config))

    def _report():
        import paper_2601_00397_b200._lib as _lib
        with open(os.environ["TWB200_LIVE_LOG"], "w") as fh:
            json.dump({"predict_calls": _calls["n"], "kinds": _calls["kinds"],
                       "native": os.path.abspath(_lib.load()._name)}, fh)

    _ref_predictor.build_predictor = build_predictor
    atexit.register(_report)
''')

# runner process: optionally the native BarrierCore inside the reference's TimekeeperServer
# (timekeeper.py:435 constructs it by module-global name); run_benchmark's verify_log then
# replays the server's log through the reference's own BarrierCore (runner.py:182)
RUNNER = textwrap.dedent('''
    import json, os, sys
    cores = []
    if os.environ.get("TWB200_NATIVE_CORE"):
        sys.path.insert(0, os.environ["TWB200_ROOT"])
        import timewarp.timekeeper as _tk
        from paper_2601_00397_b200.barrier_core import NativeBarrierCore

        class _Core(NativeBarrierCore):
            def __init__(self, *a, **k):
                super().__init__(*a, **k)
                cores.append(type(self).__mro__[1].__name__)

        _tk.BarrierCore = _Core
    from timewarp.runner import run_benchmark, run_oracle
    doc = json.loads(sys.argv[1]); out = sys.argv[2]
    rep = run_benchmark(doc, "timewarp", os.path.join(out, "live"), verify_log=True)
    run_oracle(doc, os.path.join(out, "oracle"))
    json.dump({"epoch_ns": rep.epoch_ns, "mode": rep.mode, "cores": cores},
              open(os.path.join(out, "live.json"), "w"))
''')


def _load(path):
    with open(path, encoding="utf-8") as fh:
        return [json.loads(line) for line in fh if line.strip()]


def _run_live(tmp_path, doc, device_predictor=True, native_core=False):
    site = tmp_path / "site"
    site.mkdir()
    if device_predictor:
        (site / "sitecustomize.py").write_text(SITECUSTOMIZE)
    out = tmp_path / "runs"
    out.mkdir()
    log = tmp_path / "live_log.json"
    env = dict(os.environ)
    env["TWB200_ROOT"] = ROOT
    env["TWB200_LIVE_LOG"] = str(log)
    if native_core:
        env["TWB200_NATIVE_CORE"] = "1"
    # the runner (and the oracle leg) run plain reference code; only the engine
    # subprocess's predictor factory is swapped
    runner_env = dict(env)
    runner_env["PYTHONPATH"] = REF
    engine_pp = os.pathsep.join([str(site), REF])
    runner_env["TWB200_ENGINE_PYTHONPATH"] = engine_pp
    code = ("import os, subprocess\n"
            "_popen = subprocess.Popen\n"
            "class _P(_popen):\n"
            "    def __init__(self, cmd, *a, **k):\n"
            "        if isinstance(cmd, list) and 'timewarp.engine_main' in cmd:\n"
            "            e = dict(os.environ); e['PYTHONPATH'] = os.environ['TWB200_ENGINE_PYTHONPATH']\n"
            "            k['env'] = e\n"
            "        super().__init__(cmd, *a, **k)\n"
            "subprocess.Popen = _P\n" + RUNNER)
    proc = subprocess.run([sys.executable, "-c", code, json.dumps(doc), str(out)], env=runner_env,
                          capture_output=True, text=True, timeout=900)
    if proc.returncode != 0:
        tail = ""
        err = out / "live" / "engine_stderr.log"
        if err.exists():
            tail = err.read_text()[-3000:]
        raise AssertionError(f"live run failed:\n{proc.stdout[-2000:]}\n{proc.stderr[-3000:]}\n{tail}")
    live = _load(out / "live" / "engine_events.jsonl")
    ref = _load(out / "oracle" / "engine_events.jsonl")
    meta = json.loads((out / "live.json").read_text())
    hook = json.loads(log.read_text()) if device_predictor else None
    return live, ref, meta, hook


def _assert_same(live, ref, meta):
    # pkg/tests/test_harness_integration.py:77-84
    assert [(e["request_id"], e["kind"], e["step"]) for e in live] == \
        [(e["request_id"], e["kind"], e["step"]) for e in ref]
    assert [int(e["virtual_ts_ns"]) - meta["epoch_ns"] for e in live] == \
        [int(e["virtual_ts_ns"]) for e in ref]


SMOKE = {  # pkg/tests/test_harness_integration.py:16-34
    "workload": {"source": "poisson", "qps": 8, "seed": 42, "num_requests": 10,
                 "prompt_tokens": 512, "output_tokens": 16},
    "engine": {"chunk_size": 512, "max_batch_tokens": 512, "max_running": 8,
               "kv_block_tokens": 16, "kv_capacity_blocks": 4096, "policy": "mixed"},
    "predictor": {"kind": "constant", "duration_us": 5000},
    "timekeeper": {"jitter_cooldown_us": 500},
}


@pytest.mark.gpu
def test_live_engine_constant_predictor_matches_oracle(tmp_path):
    live, ref, meta, hook = _run_live(tmp_path, SMOKE)
    assert meta["mode"] == "timewarp"
    assert len(live) == len(ref) > 0
    _assert_same(live, ref, meta)
    assert hook["kinds"] == ["constant"]
    assert hook["predict_calls"] == max(e["step"] for e in ref)
    assert hook["native"].startswith(ROOT)


TABLE_DOC = {
    "workload": {"source": "poisson", "qps": 16, "seed": 7, "num_requests": 40,
                 "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
                 "output_tokens": {"kind": "uniform", "low": 4, "high": 48}},
    "engine": {"chunk_size": 256, "max_batch_tokens": 1024, "max_running": 16,
               "kv_block_tokens": 16, "kv_capacity_blocks": 2048, "policy": "prefill_prioritized"},
    "predictor": {"kind": "table", "path": calibration.csv_path("8b", 2, 2), "allow_extrapolation": True},
    "timekeeper": {"jitter_cooldown_us": 500},
}


@pytest.mark.gpu
def test_live_engine_table_predictor_matches_oracle(tmp_path):
    doc = TABLE_DOC
    live, ref, meta, hook = _run_live(tmp_path, doc)
    assert len(live) == len(ref) > 0
    _assert_same(live, ref, meta)
    assert hook["kinds"] == ["table"]
    assert hook["predict_calls"] == max(e["step"] for e in ref)


def test_live_timekeeper_with_native_core_matches_oracle(tmp_path):
    """SURVEY §8f row 3 in the live stack (CPU: host C++ core, reference predictor): the
    reference's TimekeeperServer drives the native BarrierCore over TCP; the events equal
    the oracle's and the server log replays through the reference's BarrierCore."""
    live, ref, meta, _ = _run_live(tmp_path, TABLE_DOC, device_predictor=False, native_core=True)
    assert meta["cores"] == ["NativeBarrierCore"]
    assert len(live) == len(ref) > 0
    _assert_same(live, ref, meta)


@pytest.mark.gpu
def test_live_stack_native_core_and_device_predictor_match_oracle(tmp_path):
    live, ref, meta, hook = _run_live(tmp_path, TABLE_DOC, device_predictor=True, native_core=True)
    assert meta["cores"] == ["NativeBarrierCore"]
    _assert_same(live, ref, meta)
    assert hook["predict_calls"] == max(e["step"] for e in ref)
