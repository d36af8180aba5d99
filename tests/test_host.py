"""CPU tests: the C-ABI library's exports, host-side packing, presets, sharding (gloo)."""

import os
import re
import subprocess

import numpy as np
import pytest

from paper_2601_00397_b200._lib import TW_TABLE_HOLE

from paper_2601_00397_b200 import _lib, calibration, presets
from paper_2601_00397_b200._lib import PRED_DESC_DTYPE, PSET_HEADER_DTYPE
from paper_2601_00397_b200.predictor import (
    BatchComposition,
    DecodeSlot,
    NegativeDuration,
    PredictorError,
    PredictorSet,
    PrefillChunk,
    TableParseError,
    TablePredictor,
    build_predictor,
    pack_batches,
)
from paper_2601_00397_b200.sweep import EngineConfig, SchedulingPolicy
from paper_2601_00397_b200.timekeeper import OpStream, client_index, pack_streams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "twb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(tw_[a-z_0-9]+)\(", text, re.M)))


def test_header_declares_what_the_binding_binds():
    assert declared_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2601_00397_b200.build import build_native

        build_native()
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tw_abi_version() == _lib.ABI_VERSION
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", nm), name


def test_sass_is_sm100a_and_uses_the_bulk_copy_engine():
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UBLKCP" in out  # cp.async.bulk (TMA) staging of the predictor blob


def test_missing_library_fails_loudly(tmp_path):
    import importlib

    mod = importlib.reload(_lib)
    try:
        with pytest.raises(mod.NativeLibraryMissing):
            mod.load(str(tmp_path / "nope.so"))
    finally:
        importlib.reload(_lib)


def test_pset_blob_layout_round_trips():
    t = TablePredictor({(0, 1): 100, (512, 1): 2000, (512, 8): 3000}, allow_extrapolation=True)
    ps = PredictorSet([build_predictor({"kind": "constant", "duration_us": 7}), t,
                       build_predictor({"kind": "linear", "base_us": 1.5, "per_decode_us": 2.0})])
    blob = ps.blob
    assert blob.size % 16 == 0
    hdr = blob[:32].view(PSET_HEADER_DTYPE)[0]
    assert hdr["magic"] == _lib.TW_PSET_MAGIC and hdr["n_desc"] == 3 and hdr["total_bytes"] == blob.size
    assert hdr["version"] == 2 and hdr["core_bytes"] == hdr["fast_off"] == ps.core_nbytes
    descs = blob[32 : 32 + 3 * 64].view(PRED_DESC_DTYPE)
    assert descs["kind"].tolist() == [0, 2, 1]
    assert descs[0]["constant_us"] == 7 and descs[2]["per_decode_us"] == 2.0
    off, np_, nd = int(descs[1]["table_off"]), int(descs[1]["np"]), int(descs[1]["nd"])
    assert off % 16 == 0
    pax = blob[off : off + 4 * np_].view(np.int32)
    dax = blob[off + 4 * np_ : off + 4 * (np_ + nd)].view(np.int32)
    g0 = off + ((4 * (np_ + nd) + 7) // 8) * 8
    grid = blob[g0 : g0 + 8 * np_ * nd].view(np.int64).reshape(np_, nd)
    assert pax.tolist() == [0, 512] and dax.tolist() == [1, 8]
    assert grid.tolist() == [[100, TW_TABLE_HOLE], [2000, 3000]]


def test_predictor_construction_errors_mirror_reference(tmp_path):
    with pytest.raises(TableParseError):
        TablePredictor({})
    # negative rows are valid through the constructor (only from_csv rejects them)
    assert TablePredictor({(0, 1): -5, (8, 1): 3})._rows[(0, 1)] == -5
    with pytest.raises(NegativeDuration):
        build_predictor({"kind": "constant", "duration_us": -1})
    with pytest.raises(PredictorError):
        build_predictor({"kind": "quadratic"})
    p = tmp_path / "c.csv"
    p.write_text("total_prefill_tokens,num_decodes,duration_us\n0,1,100\n512,1,2000\n512,1,2100\n")
    t = TablePredictor.from_csv(str(p))
    assert t._rows[(512, 1)] == 2100
    p.write_text("prefill,decodes,us\n1,2,3\n")
    with pytest.raises(TableParseError):
        TablePredictor.from_csv(str(p))
    p.write_text("total_prefill_tokens,num_decodes,duration_us\n0,1,fast\n")
    with pytest.raises(TableParseError):
        TablePredictor.from_csv(str(p))
    p.write_text("total_prefill_tokens,num_decodes,duration_us\n0,1,-5\n")
    with pytest.raises(NegativeDuration):
        TablePredictor.from_csv(str(p))


def test_pack_batches_csr():
    chunky = BatchComposition(
        prefill_chunks=(PrefillChunk("r1", 256, 0), PrefillChunk("r2", 128, 512)),
        decodes=(DecodeSlot("r3", 512), DecodeSlot("r4", 700)),
    )
    off, tok, ctx = pack_batches([chunky, BatchComposition()])
    assert off.tolist() == [0, 4, 4]
    assert tok.tolist() == [256, 128, -1, -1]
    assert ctx.tolist() == [0, 512, 512, 700]


def test_engine_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        EngineConfig(chunk_size=0)
    with pytest.raises(ValueError):
        EngineConfig(chunk_size=1024, max_batch_tokens=512)
    with pytest.raises(ValueError):
        EngineConfig(kv_block_tokens=0)
    with pytest.raises(ValueError):
        EngineConfig(pp_stages=0)
    assert EngineConfig.from_doc({"policy": "prefill_prioritized"}).policy is SchedulingPolicy.PREFILL_PRIORITIZED


def test_presets_shapes():
    sw = presets.sweep_1024()
    assert len(sw) == 1024
    assert sw.workloads.n_workloads == 1 and sw.workloads.sizes().tolist() == [1000]
    assert set(sw.cfgs["pred_id"].tolist()) == set(range(8))
    assert (sw.cfgs["flags"] == 1).all() and (sw.cfgs["tk_cooldown_ns"] == 500_000).all()
    big = presets.sweep_65536(seeds=(1, 2))
    assert len(big) == 1024 * 2 * 2


def test_calibration_csvs_are_frozen():
    for m in calibration.MODELS:
        for tp, pp in calibration.TP_PP_GRID:
            t = TablePredictor.from_csv(calibration.csv_path(m, tp, pp), allow_extrapolation=True)
            assert t._rows == calibration.table_rows(m, tp, pp)
    assert calibration.table_rows("8b", 1, 1)[(0, 1)] == 835
    assert round(calibration.scale("70b", 4, 2), 2) == 6.22


def test_opstream_encoding():
    h = OpStream()
    a = h.register_actor()
    o = h.register_observer()
    h.seal()
    h.jump(a, 5)
    h.enter(a, "g", 2)
    h.enter(a, "h", 1)
    h.jump("actor99", 3)
    h.jump("bogus", 3)
    h.deregister(o)
    ops, off, wall0, cool, sup = pack_streams([h])
    assert ops["type"].tolist() == [0, 1, 2, 3, 4, 4, 7, 7, 5]  # never-issued ids are unknown clients
    assert ops["group"].tolist()[4:6] == [0, 1]
    assert ops["client"].tolist()[8] == 1
    assert client_index("observer2") == 1 and client_index("nope") == -1
    assert off.tolist() == [0, 9]


def test_opstream_only_maps_ids_the_core_issued():
    """'actor01', an observer's index under the actor prefix and registrations after the
    seal are unknown clients, as in the reference core (UnknownClient, timekeeper.py:122-128),
    checked through the C oracle's replay (ack 3 = UnknownClient, 5 = RoleViolation,
    1 = RegistrationSealed)."""
    from oracle import oracle as orc

    h = OpStream(cooldown_ns=0)
    a = h.register_actor()
    o = h.register_observer()
    h.seal()
    late = h.register_actor()
    assert (a, o, late) == ("actor1", "observer2", None)
    h.jump("actor01", 5)
    h.jump("actor2", 5)
    h.jump(o, 5)
    h.jump(a, 7)
    ops, off, wall0, cool, sup = pack_streams([h])
    assert ops["type"].tolist() == [0, 1, 2, 0, 7, 7, 3, 3]
    ack, events, fin = orc.tk_replay(ops, off, wall0, cool, sup)
    assert ack.tolist()[:8] == [0, 0, 0, 1, 3, 3, 5, 0]


def test_partition_balances_and_covers():
    from paper_2601_00397_b200.distributed import partition

    costs = np.random.default_rng(0).random(1000) * 10
    shards = partition(costs, 8)
    allids = np.sort(np.concatenate(shards))
    assert allids.tolist() == list(range(1000))
    loads = [costs[s].sum() for s in shards]
    assert max(loads) - min(loads) <= costs.max()


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2601_00397_b200._lib import SIM_RESULT_DTYPE
    from paper_2601_00397_b200.distributed import gather_results, partition

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n = 37
    shards = partition(np.arange(n, dtype=np.float64) + 1, world)
    ids = shards[rank]
    res = np.zeros(len(ids), SIM_RESULT_DTYPE)
    res["steps"] = ids * 10
    res["digest"] = ids.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    res["final_now_ns"] = ids + 1_790_000_000_000_000_000
    merged = gather_results(ids, res, n, max(len(s) for s in shards), torch.device("cpu"))
    q.put((rank, merged["steps"].tolist(), merged["final_now_ns"].tolist(), merged["digest"].tolist()))
    dist.destroy_process_group()


def test_sharded_gather_world2_gloo():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, steps, final, dig in outs:
        assert steps == [i * 10 for i in range(37)]
        assert final == [i + 1_790_000_000_000_000_000 for i in range(37)]
        assert dig == [(i * 0x9E3779B97F4A7C15) % (1 << 64) for i in range(37)]


def test_bulk_lookup_section_decodes_to_the_tables():
    """The derived bulk-lookup section (twb200.h) answers every in-range key with the
    same bracket and corners as the table itself: records by bit length give the floor
    interval, quads give the four grid corners (CPU decode of the blob the GPU reads)."""
    from _fixtures import predictor_golden

    _, preds, *_ = predictor_golden()
    ps = PredictorSet(list(preds) + list(presets.calibration_set().predictors))
    blob = ps.blob
    hdr = blob[:32].view(PSET_HEADER_DTYPE)[0]
    n = int(hdr["n_desc"])
    qh = blob[int(hdr["fast_off"]) : int(hdr["fast_off"]) + 8 * n].view(np.uint32).reshape(n, 2)
    words = blob.view(np.int32)
    rng = np.random.default_rng(3)
    n_fast = 0
    for k, p in enumerate(ps.predictors):
        tab = p._table()
        if not (int(qh[k, 1]) & _lib.TW_QHDR_FAST):
            assert tab is None or tab[2].max() >= 2**31 or tab[0][0] < 0 or tab[1][0] < 0 or \
                tab[2][tab[2] != TW_TABLE_HOLE].min() < 0
            continue
        n_fast += 1
        pax, dax, grid = tab
        grid = np.where(grid == TW_TABLE_HOLE, -1, grid)  # the int32 quads mark holes with -1
        nd = (int(qh[k, 1]) >> 16) & 0x7FFF
        assert nd == len(dax)
        quads = int(qh[k, 0]) & 0xFFFF
        recs = {"p": int(qh[k, 0]) >> 16, "d": int(qh[k, 1]) & 0xFFFF}

        def look(which, v):
            r = words[(recs[which] + int(v).bit_length()) * 4 :][:3]
            return int(r[0]), int(r[1]), int(r[2])

        qp = np.concatenate([pax, pax + 1, pax - 1, rng.integers(0, int(pax[-1]) + 2, 200)])
        qd = np.concatenate([dax, dax + 1, dax - 1, rng.integers(0, int(dax[-1]) + 2, 200)])
        for which, axis, qs in (("p", pax, qp), ("d", dax, qd)):
            for v in qs[qs >= 0]:
                lo, hi, info = look(which, v)
                inside = axis[0] <= v <= axis[-1]
                if info < 0:
                    continue  # the bucket straddles several intervals: generic path
                if not (lo <= v <= hi):
                    assert not inside
                    continue
                assert inside
                i = int(np.searchsorted(axis, v, side="right")) - 1
                assert (info, lo) == (i, int(axis[i]))
                assert hi == (int(axis[i + 1]) if i + 1 < len(axis) else int(axis[i]))
        for i in range(len(pax)):
            for j in range(len(dax)):
                q = words[(quads * 16) // 4 + 4 * (i * nd + j) :][:4]
                i1, j1 = min(i + 1, len(pax) - 1), min(j + 1, len(dax) - 1)
                assert q.tolist() == [grid[i, j], grid[i1, j], grid[i, j1], grid[i1, j1]]
    assert n_fast >= 16
    assert int(hdr["n_axis_sets"]) < 2 * n_fast  # calibration tables share their axes


def test_ziggurat_tables_and_numpy_draw_restatement():
    """csrc/ziggurat_tables.h holds the installed numpy's tables, and the restated draw
    algorithms (oracle/numpy_rng.py, the basis of csrc/workload.cu) reproduce numpy's
    Generator.exponential / integers streams exactly, slow paths included."""
    import importlib.util
    import re as _re

    spec = importlib.util.spec_from_file_location("gen_zig", os.path.join(ROOT, "scripts", "gen_ziggurat.py"))
    gz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gz)
    ke, we, fe = gz.locate()
    text = open(os.path.join(ROOT, "paper_2601_00397_b200", "csrc", "ziggurat_tables.h")).read()
    blocks = _re.findall(r"\{([^}]*)\}", text)
    assert [int(v, 16) for v in _re.findall(r"0x[0-9a-f]+", blocks[0])] == list(ke)
    assert [float(v) for v in blocks[1].replace("\n", "").split(",") if v.strip()] == list(we)
    assert [float(v) for v in blocks[2].replace("\n", "").split(",") if v.strip()] == list(fe)

    from oracle.numpy_rng import Pcg64, integers_closed, standard_exponential

    n = 0
    for seed in (1, 7, 99, 2601):
        rng = np.random.default_rng(seed)
        g = Pcg64(rng.bit_generator.state)
        for i in range(2500):
            assert rng.exponential(0.25) == 0.25 * standard_exponential(g, ke, we, fe)
            lo, hi = [(64, 2048), (1, 1), (0, 2**31 - 1), (5, 6)][i % 4]
            assert int(rng.integers(lo, hi + 1)) == integers_closed(g, lo, hi)
            n += 1
    assert n == 10_000


def test_c_abi_rejects_bad_arguments_before_touching_the_device():
    """The boundary's error behaviour (twb200.h): invalid pointers, sizes and blobs return
    TW_EINVAL with a message naming the entry point, before any CUDA call (so this runs
    without a GPU), and a zero-sized request is a successful no-op."""
    import ctypes

    from paper_2601_00397_b200 import _lib

    lib = _lib.load()
    V = ctypes.c_void_p
    null = V(0)
    blob = (ctypes.c_uint8 * 64)()  # 16-B aligned enough for the size check, but no valid header

    def err():
        return lib.tw_last_error().decode()

    cases = [
        ("tw_sim_many", lambda: lib.tw_sim_many(null, 0, null, 1, null, null, null, null, null, null, null, null,
                                                 null, null, null, 256, null, 0, null)),
        ("tw_predict_features", lambda: lib.tw_predict_features(null, 64, null, null, null, null, 10, null, null)),
        ("tw_predict_batches", lambda: lib.tw_predict_batches(ctypes.cast(blob, V), 64, null, null, null, null, 5,
                                                               null, null, null)),
        ("tw_metrics_many", lambda: lib.tw_metrics_many(null, 3, null, null, null, null, null, null, null, null,
                                                         1000, null, 0, null, null)),
        ("tw_generate_poisson", lambda: lib.tw_generate_poisson(null, 4, null, null, null, null, null, null)),
        ("tw_predict_one_sync", lambda: lib.tw_predict_one_sync(null, 64, null, 3, 0, null, 0, null, null)),
    ]
    for name, call in cases:
        rc = call()
        assert rc == _lib.TW_EINVAL, (name, rc, err())
        msg = err()
        assert msg and (name in msg or "pset" in msg), (name, msg)
    # empty requests are no-ops that never reach the device
    assert lib.tw_generate_poisson(null, 0, null, null, null, null, null, null) == _lib.TW_OK
    assert lib.tw_metrics_many(null, 0, null, null, null, null, null, null, null, null, 1000, null, 0, null,
                               null) == _lib.TW_OK


def test_exceptions_derive_from_the_host_frameworks_when_present():
    """With the reference package importable (baseline/_ref), host code that catches
    timewarp's exception classes catches this engine's (drop-in error behaviour)."""
    import subprocess
    import sys

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "timewarp")):
        pytest.skip("reference not installed under baseline/_ref")
    code = (
        "import timewarp.predictor as hp, timewarp.oracle as ho, timewarp.workload as hw\n"
        "from paper_2601_00397_b200 import predictor as p, sweep as s, workload as w\n"
        "pairs = [(p.PredictorError, hp.PredictorError), (p.EmptyBatch, hp.EmptyBatch),\n"
        "         (p.NegativeDuration, hp.NegativeDuration), (p.TableMiss, hp.TableMiss),\n"
        "         (p.TableParseError, hp.TableParseError), (p.TableMiss, hp.PredictorError),\n"
        "         (s.OracleStalled, ho.OracleStalled), (w.WorkloadError, hw.WorkloadError),\n"
        "         (w.TraceParseError, hw.TraceParseError), (w.TraceParseError, hw.WorkloadError)]\n"
        "assert all(issubclass(a, b) for a, b in pairs)\n"
        "try:\n    p.TablePredictor({})\nexcept hp.TableParseError:\n    print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ref, ROOT]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]


def test_standalone_workload_schema_equals_the_reference(tmp_path):
    """Without the host framework importable, workload.py declares the schema itself: it must
    parse, render, fingerprint, draw and load traces exactly like timewarp.workload
    (baseline/_ref), including the error texts."""
    import importlib
    import sys

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "timewarp")):
        pytest.skip("reference not installed under baseline/_ref")
    from paper_2601_00397_b200 import workload as ours

    assert ours._HOST is None  # standalone in the test process
    sys.path.insert(0, ref_dir)
    try:
        ref = importlib.import_module("timewarp.workload")
    finally:
        sys.path.remove(ref_dir)
    docs = [{"source": "poisson", "qps": 8, "seed": 3, "num_requests": 50,
             "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048}, "output_tokens": 17},
            {"qps": 2.5, "seed": 9, "num_requests": 20, "prompt_tokens": {"value": 300},
             "output_tokens": {"kind": "uniform", "low": 1, "high": 4}}, {}]
    for doc in docs:
        a, b = ours.WorkloadSpec.from_doc(doc), ref.WorkloadSpec.from_doc(doc)
        assert a.to_doc() == b.to_doc() and a.fingerprint() == b.fingerprint()
        if a.num_requests:
            assert [tuple(vars(x).values()) for x in ours.generate_arrivals(a)] == \
                   [tuple(vars(x).values()) for x in ref.generate_arrivals(b)]
    for bad in ({"kind": "zipf"},):
        with pytest.raises(Exception) as e1:
            ours.TokenDist.from_doc(bad)
        with pytest.raises(Exception) as e2:
            ref.TokenDist.from_doc(bad)
        assert str(e1.value) == str(e2.value)
    good = tmp_path / "t.csv"
    good.write_text("prompt_tokens,arrival_ms,output_tokens,extra\n10,5.5,3,x\n20,1.25,4,y\n7,5.5,1,z\n")
    assert [tuple(vars(x).values()) for x in ours.load_trace(str(good))] == \
           [tuple(vars(x).values()) for x in ref.load_trace(str(good))]
    for text in ("arrival_ms,prompt_tokens\n1,2\n", "arrival_ms,prompt_tokens,output_tokens\n1,x,2\n",
                 "arrival_ms,prompt_tokens,output_tokens\n-1,2,2\n"):
        bad = tmp_path / "b.csv"
        bad.write_text(text)
        with pytest.raises(Exception) as e1:
            ours.load_trace(str(bad))
        with pytest.raises(Exception) as e2:
            ref.load_trace(str(bad))
        assert str(e1.value) == str(e2.value) and type(e1.value).__name__ == type(e2.value).__name__
