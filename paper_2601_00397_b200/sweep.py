"""Bulk emulation of many serving configurations — the B200 event loop's host side.

Mirrors the reference's event-loop interfaces (pkg/src/timewarp/oracle.py:49-54 and
pkg/src/timewarp/engine.py:46-133):

* :func:`simulate` is a drop-in for ``timewarp.oracle.simulate``: same arguments,
  same ``[{"request_id", "kind", "virtual_ts_ns", "step"}]`` result, raises
  :class:`OracleStalled` on a stall — but the loop runs in libtwb200's sm_100a
  kernel (one warp, full event dump).
* :func:`simulate_many` / :class:`DeviceSweep` run thousands of configs in one
  persistent launch and return fixed-size per-config records (steps, virtual span,
  event digest, Timekeeper state, status) plus optional per-request FIRST_TOKEN /
  FINISHED stamps and audited full event streams.
* :meth:`DeviceSweep.run_metrics` reduces those stamps on device to each config's
  ``RunReport.summary()`` numbers (metrics.py:38-253): TTFT / e2e / TPOT nearest-rank
  p50/p90/p99 and means, output tokens, virtual span, tokens per virtual second;
  :func:`summary_doc` renders one record in the reference's summary layout.
"""

from __future__ import annotations

import enum
import json
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._host import host_bases
from ._lib import (
    EVENT_DTYPE,
    RUN_METRICS_DTYPE,
    TW_METRICS_INCOMPLETE,
    TW_METRICS_OK,
    EVENT_KIND_NAMES,
    SIM_CFG_DTYPE,
    SIM_RESULT_DTYPE,
    TW_SIM_BAD_CONFIG,
    TW_SIM_CAPACITY,
    TW_SIM_OK,
    TW_SIM_OVERFLOW_BIT,
    TW_SIM_PRED_ERROR,
    TW_SIM_STALLED_ACTIVE,
    TW_SIM_STALLED_KV,
    TW_SIM_TIMEKEEPER,
)
from .predictor import (
    ConstantPredictor,
    LinearPredictor,
    PredictorSet,
    TablePredictor,
    raise_for_code,
)
from .workload import PackedWorkloads, pack_arrivals

DEFAULT_COOLDOWN_NS = 500_000  # timekeeper.py:36 (DEFAULT_COOLDOWN_US * NS_PER_US)


class SchedulingPolicy(enum.Enum):
    MIXED = "mixed"
    PREFILL_PRIORITIZED = "prefill_prioritized"


class EngineError(Exception):
    pass


class OracleStalled(*(host_bases("oracle", "OracleStalled") or (Exception,))):  # oracle.py:26
    """The simulated engine can never make progress again (oracle.py:26-27)."""


@dataclass(frozen=True)
class EngineConfig:
    """Same fields, defaults and validation as engine.py:98-133."""

    chunk_size: int = 512
    policy: SchedulingPolicy = SchedulingPolicy.MIXED
    max_batch_tokens: int = 512
    max_running: int = 256
    kv_block_tokens: int = 16
    kv_capacity_blocks: int = 4096
    workers_per_replica: int = 1
    pp_stages: int = 1

    def __post_init__(self) -> None:
        if self.chunk_size < 1:
            raise ValueError(f"chunk_size must be >= 1, got {self.chunk_size}")
        if self.max_batch_tokens < self.chunk_size:
            raise ValueError(
                f"max_batch_tokens ({self.max_batch_tokens}) must be >= chunk_size ({self.chunk_size})"
            )
        if self.kv_block_tokens < 1 or self.kv_capacity_blocks < 1:
            raise ValueError("KV geometry must be positive")
        if self.workers_per_replica < 1 or self.pp_stages < 1:
            raise ValueError("worker grid dimensions must be >= 1")

    @classmethod
    def from_doc(cls, doc: dict) -> "EngineConfig":
        return cls(
            chunk_size=int(doc.get("chunk_size", 512)),
            policy=SchedulingPolicy(doc.get("policy", "mixed")),
            max_batch_tokens=int(doc.get("max_batch_tokens", 512)),
            max_running=int(doc.get("max_running", 256)),
            kv_block_tokens=int(doc.get("kv_block_tokens", 16)),
            kv_capacity_blocks=int(doc.get("kv_capacity_blocks", 4096)),
            workers_per_replica=int(doc.get("workers_per_replica", 1)),
            pp_stages=int(doc.get("pp_stages", 1)),
        )


def _policy_code(policy) -> int:
    value = getattr(policy, "value", policy)
    if value == "mixed":
        return _lib.TW_POLICY_MIXED
    if value == "prefill_prioritized":
        return _lib.TW_POLICY_PREFILL_PRIORITIZED
    raise ValueError(f"unknown scheduling policy {policy!r}")


@dataclass
class SweepConfig:
    """One emulated configuration: engine knobs + which predictor and workload it uses."""

    engine: object  # EngineConfig (ours or the reference's: duck-typed)
    pred_id: int = 0
    workload_id: int = 0
    epoch_ns: int = 0
    timekeeper: bool = True
    tk_cooldown_ns: int = DEFAULT_COOLDOWN_NS
    label: dict = field(default_factory=dict)


def config_array(configs: Sequence[SweepConfig]) -> np.ndarray:
    a = np.zeros(len(configs), SIM_CFG_DTYPE)
    for i, c in enumerate(configs):
        e = c.engine
        a[i]["chunk_size"] = e.chunk_size
        a[i]["max_batch_tokens"] = e.max_batch_tokens
        a[i]["max_running"] = e.max_running
        a[i]["kv_block_tokens"] = e.kv_block_tokens
        a[i]["kv_capacity_blocks"] = e.kv_capacity_blocks
        a[i]["workers_per_replica"] = e.workers_per_replica
        a[i]["pp_stages"] = e.pp_stages
        a[i]["policy"] = _policy_code(e.policy)
        a[i]["pred_id"] = c.pred_id
        a[i]["workload_id"] = c.workload_id
        a[i]["epoch_ns"] = c.epoch_ns
        a[i]["tk_cooldown_ns"] = c.tk_cooldown_ns
        a[i]["flags"] = TW_SIM_TIMEKEEPER if c.timekeeper else 0
    return a


def as_device_predictor(p):
    """Accept our predictors or the reference's (duck-typed by their attributes)."""
    if isinstance(p, (ConstantPredictor, LinearPredictor, TablePredictor)):
        return p
    if hasattr(p, "_rows") and hasattr(p, "allow_extrapolation"):
        return TablePredictor(p._rows, allow_extrapolation=p.allow_extrapolation)
    if hasattr(p, "per_prefill_token_us"):
        return LinearPredictor(p.base_us, p.per_prefill_token_us, p.per_decode_us, p.per_context_token_us)
    if hasattr(p, "duration_us"):
        return ConstantPredictor(p.duration_us)
    raise TypeError(f"cannot run predictor {type(p).__name__} on the B200 engine")


COST_MODEL_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cost_model.json")


def cost_features(pset: PredictorSet, cfgs: np.ndarray, wl: PackedWorkloads):
    """Numeric per-config features of the event loop's cost (log scale where multiplicative)."""
    out_tok = np.ones(wl.n_workloads, np.float64)
    prm_tok = np.ones(wl.n_workloads, np.float64)
    for w in range(wl.n_workloads):
        lo, hi = int(wl.wl_off[w]), int(wl.wl_off[w + 1])
        out_tok[w] = float(wl.output[lo:hi].astype(np.int64).sum()) + 1.0
        prm_tok[w] = float(wl.prompt[lo:hi].astype(np.int64).sum()) + 1.0
    step_us = np.ones(len(pset.predictors))
    for i, p in enumerate(pset.predictors):
        if isinstance(p, ConstantPredictor):
            step_us[i] = max(p.duration_us, 1)
        elif isinstance(p, LinearPredictor):
            step_us[i] = max(abs(p.base_us) + abs(p.per_decode_us), 1.0)
        else:
            step_us[i] = max(min(p._rows.values()), 1)
    pid = np.clip(cfgs["pred_id"], 0, len(step_us) - 1)
    wid = cfgs["workload_id"]
    names = ["chunk", "mbt", "max_running", "tp", "pp", "policy", "step_us", "out_tokens", "prompt_tokens"]
    F = np.stack([
        np.log2(np.maximum(cfgs["chunk_size"], 1)), np.log2(np.maximum(cfgs["max_batch_tokens"], 1)),
        np.log2(np.maximum(cfgs["max_running"], 1)), np.log2(np.maximum(cfgs["workers_per_replica"], 1)),
        cfgs["pp_stages"].astype(np.float64), cfgs["policy"].astype(np.float64), np.log(step_us[pid]),
        np.log(out_tok[wid]), np.log(prm_tok[wid]),
    ], 1)
    return names, F


def cost_design(names, F):
    """Design matrix of the cost model: 1, the features, and their pairwise products."""
    cols, terms = [np.ones(len(F))], ["1"]
    for i, a in enumerate(names):
        cols.append(F[:, i])
        terms.append(a)
    for i in range(len(names)):
        for j in range(i, len(names)):
            cols.append(F[:, i] * F[:, j])
            terms.append(f"{names[i]}*{names[j]}")
    return np.stack(cols, 1), terms


_COST_MODEL = None


def estimate_cost(pset: PredictorSet, cfgs: np.ndarray, wl: PackedWorkloads) -> np.ndarray:
    """Relative cost per config (~ device cycles), for the LPT shard partition and the
    largest-first pull order: a log-linear model with pairwise terms fitted to measured
    per-config cycles of config 5 (cost_model.json, refit by scripts/fit_cost.py)."""
    global _COST_MODEL
    if len(cfgs) == 0:
        return np.zeros(0)
    if _COST_MODEL is None:
        with open(COST_MODEL_PATH) as fh:
            _COST_MODEL = json.load(fh)
    names, F = cost_features(pset, cfgs, wl)
    if names != _COST_MODEL["features"]:
        raise EngineError("cost_model.json was fitted on other features; rerun scripts/fit_cost.py")
    X, _ = cost_design(names, F)
    return np.exp(np.clip(X @ np.asarray(_COST_MODEL["coef"]), -700, 700))


@dataclass
class SweepResult:
    results: np.ndarray  # SIM_RESULT_DTYPE per config
    first_ns: np.ndarray | None = None  # int64 per (config, request) at req_base[c] + i
    finish_ns: np.ndarray | None = None
    req_base: np.ndarray | None = None
    events: dict = field(default_factory=dict)  # config -> EVENT_DTYPE array (audited)
    kernel_ms: float | None = None

    @property
    def predictions(self) -> int:
        return int(self.results["steps"].sum())

    def virtual_seconds(self, epochs: np.ndarray | None = None) -> float:
        """Sum over configs of (last FINISHED ts - epoch) (metrics.py:245)."""
        end = self.results["final_now_ns"].astype(np.float64)
        if epochs is not None:
            end = end - epochs.astype(np.float64)
        return float(end.sum()) / 1e9

    def ok(self) -> np.ndarray:
        return self.results["status"] == TW_SIM_OK


class DeviceSweep:
    """All inputs and outputs of a sweep resident in HBM; ``run()`` is one launch."""

    def __init__(
        self,
        pset: PredictorSet,
        workloads: PackedWorkloads,
        cfgs: np.ndarray,
        device=None,
        per_request: bool = True,
        audit: Sequence[int] = (),
        order: np.ndarray | None = None,
    ) -> None:
        import torch

        from ._device import require_cuda, to_device

        self.device = require_cuda(device)
        self.pset = pset
        self.workloads = workloads
        self.cfgs = np.ascontiguousarray(cfgs)
        self.n_cfg = len(cfgs)
        if order is None:
            order = np.argsort(-estimate_cost(pset, self.cfgs, workloads), kind="stable").astype(np.int32)
        self.order = np.ascontiguousarray(order, np.int32)
        sizes = workloads.sizes()[self.cfgs["workload_id"]] if self.n_cfg else np.zeros(0, np.int64)
        self.req_base = np.zeros(self.n_cfg + 1, np.int64)
        np.cumsum(sizes, out=self.req_base[1:])
        # The whole blob: prediction-cache misses use its bulk-lookup section, staged in
        # shared memory by the latency variant (<= 8 configs per SM) or read from global
        # memory by the throughput variant (twb200.h, tw_sim_many).
        self.stage_bytes = pset.nbytes
        self.slot_capacity = int(max(32, int(self.cfgs["max_running"].max()) if self.n_cfg else 32))
        # up to 4096 the slot state lives in shared memory, above it in d_scratch (sim_big.cu)
        dev = self.device
        self.d_pset = pset.device_blob(dev)
        self.d_cfgs = to_device(self.cfgs, dev)
        self.d_order = to_device(self.order, dev)
        self.d_wl_off = to_device(workloads.wl_off, dev)
        self.d_ts = to_device(workloads.offset_ns, dev)
        self.d_prompt = to_device(workloads.prompt, dev)
        self.d_output = to_device(workloads.output, dev)
        self.d_res = torch.zeros(self.n_cfg * SIM_RESULT_DTYPE.itemsize + 16, dtype=torch.uint8, device=dev)
        total_req = int(self.req_base[-1])
        lib = _lib.load()
        scratch = int(lib.tw_sim_scratch_bytes(self.n_cfg, self.slot_capacity)) if self.n_cfg else 64
        # latency regime: records of the busy-period segments (tw_sim_seg_scratch_bytes; the
        # library picks them when req_base is passed, i.e. with per-request stamps)
        if per_request and self.n_cfg and not audit:
            seg = int(lib.tw_sim_seg_scratch_bytes(self.n_cfg, total_req))
            # bounded: past a quarter of free device memory the serial loop runs instead (the
            # library falls back to it when the scratch is too small for the segments)
            free, _ = torch.cuda.mem_get_info(self.device)
            if seg <= free // 4:
                scratch = max(scratch, seg)
        self.d_scratch = torch.zeros(max(64, scratch), dtype=torch.uint8, device=dev)
        self.per_request = per_request
        if per_request:
            self.d_req_base = to_device(self.req_base, dev)
            self.d_first = torch.full((max(total_req, 1),), -1, dtype=torch.int64, device=dev)
            self.d_finish = torch.full((max(total_req, 1),), -1, dtype=torch.int64, device=dev)
        else:
            self.d_req_base = self.d_first = self.d_finish = None
        self.audit = [int(c) for c in audit]
        if self.audit:
            caps = np.zeros(self.n_cfg, np.int64)
            for c in self.audit:
                lo, hi = workloads.wl_off[self.cfgs[c]["workload_id"]], workloads.wl_off[self.cfgs[c]["workload_id"] + 1]
                # at most max(output, 1) + 1 events per request: FIRST_TOKEN, output - 1
                # OUTPUT_TOKENs, FINISHED; a request with output <= 0 still emits
                # FIRST_TOKEN + FINISHED (oracle.py:93-100)
                caps[c] = int(np.maximum(workloads.output[lo:hi].astype(np.int64), 1).sum() + (hi - lo))
            self.ev_off = np.zeros(self.n_cfg + 1, np.int64)
            np.cumsum(caps, out=self.ev_off[1:])
            self.d_ev_off = to_device(self.ev_off, dev)
            self.d_ev = torch.zeros(max(int(self.ev_off[-1]), 1) * EVENT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        else:
            self.ev_off = None
            self.d_ev_off = self.d_ev = None

    @property
    def h2d_bytes(self) -> int:
        n = self.stage_bytes + self.cfgs.nbytes + self.order.nbytes + self.workloads.nbytes
        if self.per_request:
            n += self.req_base.nbytes
        return int(n)

    def run(self, stream=None) -> None:
        from ._device import ptr, stream_handle

        rc = _lib.load().tw_sim_many(
            self.d_pset.data_ptr(), self.stage_bytes, self.d_cfgs.data_ptr(), self.n_cfg,
            self.d_order.data_ptr(), self.d_wl_off.data_ptr(), self.d_ts.data_ptr(),
            self.d_prompt.data_ptr(), self.d_output.data_ptr(), self.d_res.data_ptr(),
            ptr(self.d_req_base), ptr(self.d_first), ptr(self.d_finish), ptr(self.d_ev_off),
            ptr(self.d_ev), self.slot_capacity, self.d_scratch.data_ptr(), self.d_scratch.numel(),
            stream_handle(stream),
        )
        _lib.check(rc, "tw_sim_many")

    CHECK_NAMES = ("iterations", "time_went_back", "slot_overrun", "kv_counter_diverged", "tk_went_back",
                   "tk_virtual_inconsistent", "tk_bcast_after_wall", "event_count")

    def run_checked(self, stream=None) -> np.ndarray:
        """One launch of the invariant-checking build of the event loop (tw_sim_set_checks,
        sim_check.cu): the same results, plus int32 [n_cfg, 8] counters (CHECK_NAMES;
        every column but the first must be 0). Debug path, not timed."""
        import torch

        cnt = torch.zeros(max(self.n_cfg, 1) * 8, dtype=torch.int32, device=self.device)
        lib = _lib.load()
        lib.tw_sim_set_checks(cnt.data_ptr())
        try:
            self.run(stream)
            torch.cuda.synchronize(self.device)
        finally:
            lib.tw_sim_set_checks(None)
        return cnt[: 8 * self.n_cfg].view(self.n_cfg, 8).cpu().numpy()

    # -- per-config latency summary (metrics.py:173-253) ---------------------------
    def run_metrics(self, stream=None) -> None:
        """Launch the on-device reduction of this sweep's stamps (needs per_request)."""
        import torch

        from ._device import stream_handle, to_device

        if not self.per_request:
            raise EngineError("run_metrics needs per-request stamps (DeviceSweep(per_request=True))")
        if getattr(self, "d_metrics", None) is None:
            self.d_metrics = torch.zeros(max(self.n_cfg, 1) * RUN_METRICS_DTYPE.itemsize, dtype=torch.uint8,
                                         device=self.device)
            ci = self.workloads.caller_index
            self.d_sum_order = to_device(ci, self.device) if ci is not None and len(ci) else None
            self.max_requests = int(self.workloads.sizes().max()) if self.workloads.n_workloads else 0
            # workloads above what shared memory holds keep their keys in global scratch
            nbytes = int(_lib.load().tw_metrics_scratch_bytes(self.n_cfg, self.max_requests))
            self.d_met_scratch = torch.empty(nbytes, dtype=torch.uint8, device=self.device) if nbytes else None
        sc = self.d_met_scratch
        rc = _lib.load().tw_metrics_many(
            self.d_cfgs.data_ptr(), self.n_cfg, self.d_wl_off.data_ptr(), self.d_ts.data_ptr(),
            self.d_output.data_ptr(), self.d_req_base.data_ptr(), self.d_first.data_ptr(),
            self.d_finish.data_ptr(), self.d_res.data_ptr(),
            self.d_sum_order.data_ptr() if self.d_sum_order is not None else None, self.max_requests,
            sc.data_ptr() if sc is not None else None, sc.numel() if sc is not None else 0,
            self.d_metrics.data_ptr(), stream_handle(stream),
        )
        _lib.check(rc, "tw_metrics_many")

    def fetch_metrics(self) -> np.ndarray:
        from ._device import to_numpy_struct

        return to_numpy_struct(self.d_metrics, RUN_METRICS_DTYPE, self.n_cfg)

    def fetch(self) -> SweepResult:
        from ._device import to_numpy_struct

        res = to_numpy_struct(self.d_res, SIM_RESULT_DTYPE, self.n_cfg)
        out = SweepResult(results=res, req_base=self.req_base)
        if self.per_request:
            n = int(self.req_base[-1])
            out.first_ns = self.d_first[:n].cpu().numpy()
            out.finish_ns = self.d_finish[:n].cpu().numpy()
        if self.audit:
            evs = to_numpy_struct(self.d_ev, EVENT_DTYPE, int(self.ev_off[-1]))
            for c in self.audit:
                if int(res[c]["status"]) & TW_SIM_OVERFLOW_BIT:
                    raise EngineError(f"config {c}: event dump overflowed its buffer ({int(res[c]['events'])} events)")
                k = min(int(res[c]["events"]), int(self.ev_off[c + 1] - self.ev_off[c]))
                out.events[c] = evs[self.ev_off[c] : self.ev_off[c] + k]
        return out


def simulate_many(
    workloads,
    configs: Sequence[SweepConfig],
    predictors,
    audit: Sequence[int] = (),
    per_request: bool = True,
    device=None,
) -> SweepResult:
    """Run every config's event loop on the GPU (one persistent launch).

    workloads: PackedWorkloads or a list of Arrival lists; predictors: a PredictorSet
    or a list of predictor objects (indexed by SweepConfig.pred_id).
    """
    import torch

    wl = workloads if isinstance(workloads, PackedWorkloads) else pack_arrivals(workloads)
    pset = predictors if isinstance(predictors, PredictorSet) else PredictorSet(
        [as_device_predictor(p) for p in predictors]
    )
    sweep = DeviceSweep(pset, wl, config_array(configs), device=device, per_request=per_request, audit=audit)
    sweep.run()
    torch.cuda.synchronize(sweep.device)
    return sweep.fetch()


def summary_doc(rec, mode: str = "oracle", workload_fingerprint: str = "", wall_elapsed_ns: int = 0) -> dict:
    """One RUN_METRICS_DTYPE record in RunReport.summary()'s layout (metrics.py:97-124)."""
    from .workload import NS_PER_S

    st = int(rec["status"])
    if st == TW_METRICS_INCOMPLETE:
        raise EngineError(f"IncompleteLog: {int(rec['n_missing'])} requests never finished")
    if st != TW_METRICS_OK:
        raise EngineError(f"metrics status {st}")
    ve = int(rec["virtual_elapsed_ns"])
    doc = {
        "mode": mode,
        "workload_fingerprint": workload_fingerprint,
        "num_requests": int(rec["num_requests"]),
        "virtual_elapsed_ns": ve,
        "wall_elapsed_ns": wall_elapsed_ns,
        "speedup": ve / wall_elapsed_ns if wall_elapsed_ns > 0 else float("inf"),
        "output_tokens": int(rec["output_tokens"]),
    }

    def stats(s):
        return {"p50": float(s["p50"]), "p90": float(s["p90"]), "p99": float(s["p99"]),
                "mean": float(s["mean"]), "count": int(s["count"])}

    if int(rec["num_requests"]) > 0:
        doc["ttft_ns"] = stats(rec["ttft"])
        doc["e2e_ns"] = stats(rec["e2e"])
        doc["tokens_per_virtual_s"] = float(rec["tokens_per_virtual_s"]) if ve / NS_PER_S > 0 else 0.0
    if int(rec["tpot"]["count"]) > 0:
        doc["tpot_ns"] = stats(rec["tpot"])
    return doc


def _raise_status(res, what: str = "", audited: bool = False) -> None:
    if audited and int(res["status"]) & TW_SIM_OVERFLOW_BIT:
        raise EngineError(f"{what}event dump overflowed its buffer: {int(res['events'])} events")
    st = int(res["status"]) & ~TW_SIM_OVERFLOW_BIT
    if st == TW_SIM_OK:
        return
    if st == TW_SIM_STALLED_ACTIVE:
        raise OracleStalled(f"{what}active requests with no schedulable work: KV pool cannot cover the in-flight set")
    if st == TW_SIM_STALLED_KV:
        raise OracleStalled(f"{what}queue head needs more KV blocks than the pool holds")
    if st == TW_SIM_PRED_ERROR:
        raise_for_code(int(res["pred_code"]))
    if st == TW_SIM_BAD_CONFIG:
        raise ValueError(f"{what}invalid engine config")
    if st == TW_SIM_CAPACITY:
        raise EngineError(f"{what}config exceeds the engine's slot or actor capacity")
    raise EngineError(f"{what}simulation status {st}")


def events_to_docs(ev: np.ndarray, request_ids: Sequence[str]) -> list[dict]:
    rk = ev["req_kind"].astype(np.int64)
    req = rk >> 2
    kind = rk & 3
    return [
        {
            "request_id": request_ids[int(r)],
            "kind": EVENT_KIND_NAMES[int(k)],
            "virtual_ts_ns": int(t),
            "step": int(s),
        }
        for r, k, t, s in zip(req, kind, ev["ts_ns"], ev["step"])
    ]


def simulate(arrivals, cfg, predictor, epoch_ns: int = 0) -> list[dict]:
    """Drop-in for ``timewarp.oracle.simulate`` (oracle.py:49-114), run on the GPU."""
    wl = pack_arrivals([arrivals])
    sc = SweepConfig(engine=cfg, pred_id=0, workload_id=0, epoch_ns=epoch_ns, timekeeper=False)
    out = simulate_many(wl, [sc], [predictor], audit=[0], per_request=False)
    _raise_status(out.results[0], audited=True)
    return events_to_docs(out.events[0], wl.request_ids[0])


class HostSweep(DeviceSweep):
    """A sweep driven from HOST buffers: every ``run_from_host()`` copies the inputs
    from pinned host memory to HBM and runs the event-loop kernel, all stream-ordered,
    and leaves the result records and per-request stamps in pinned host memory. This is
    the end-to-end path a host caller pays for (bench.py ``e2e``). Two output modes:

    * ``zero_copy`` (default up to 256 MB of outputs): the kernel stores records and
      stamps straight into pinned host memory over PCIe as it produces them (UVA), so
      nothing follows the kernel (config 4, 16 MB of stamps: 7.98 vs 8.3 ms per step
      with a copy after it);
    * streamed (above that; config 5 has 1 GB of stamps): the configs are laid out in
      their pull order (largest estimated cost first), so they finish roughly in stamp
      order; the kernel writes each config's record into pinned memory after a
      system-scope fence, and the host watches the records and copies each finished
      prefix of the stamps on a second stream while the kernel still runs. Only the
      last configs' stamps are copied after it.

    Records and stamps are returned in the caller's config order (``host_results``,
    ``host_stamps``)."""

    ZERO_COPY_MAX_BYTES = 256 << 20
    STREAM_CHUNK_CONFIGS = 4096  # copy granularity of the streamed mode

    def __init__(self, pset, workloads, cfgs, *args, zero_copy: bool | None = None, **kwargs) -> None:
        import torch

        cfgs = np.ascontiguousarray(cfgs)
        n_req = int(workloads.sizes()[cfgs["workload_id"]].sum()) if len(cfgs) else 0
        per_request = kwargs.get("per_request", True)
        if zero_copy is None:
            zero_copy = 64 * len(cfgs) + (16 * n_req if per_request else 0) <= self.ZERO_COPY_MAX_BYTES
        self.zero_copy = bool(zero_copy)
        self.streamed = not self.zero_copy and per_request
        self.perm = None
        if self.streamed:
            # configs in pull order: the kernel then pulls them in stamp order (order = identity)
            order = kwargs.pop("order", None)
            if order is None:
                order = np.argsort(-estimate_cost(pset, cfgs, workloads), kind="stable")
            self.perm = np.asarray(order, np.int64)  # pull index -> caller's config index
            cfgs = cfgs[self.perm]
            kwargs["order"] = np.arange(len(cfgs), dtype=np.int32)
        super().__init__(pset, workloads, cfgs, *args, **kwargs)
        self._pairs_in = []
        staged = self.d_pset[: self.stage_bytes]  # what the event loop reads of the blob
        for d in (staged, self.d_cfgs, self.d_order, self.d_wl_off, self.d_ts, self.d_prompt, self.d_output):
            h = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
            h.copy_(d.cpu())
            self._pairs_in.append((d, h))
        if self.per_request:
            h = torch.empty(self.d_req_base.shape, dtype=self.d_req_base.dtype, pin_memory=True)
            h.copy_(self.d_req_base.cpu())
            self._pairs_in.append((self.d_req_base, h))
        self._pairs_out = [(self.d_res, torch.empty(self.d_res.shape, dtype=self.d_res.dtype, pin_memory=True))]
        if self.per_request:
            for d in (self.d_first, self.d_finish):
                self._pairs_out.append((d, torch.full(d.shape, -1, dtype=d.dtype, pin_memory=True)))
        if self.zero_copy or self.streamed:  # records straight into pinned memory
            self.d_res = self._pairs_out[0][1]
        if self.zero_copy and self.per_request:  # stamps too
            self.d_first, self.d_finish = self._pairs_out[1][1], self._pairs_out[2][1]
        if self.streamed:
            raw = self._pairs_out[0][1].numpy().view(np.uint8)[: self.n_cfg * SIM_RESULT_DTYPE.itemsize]
            self._rec_view = raw.view(SIM_RESULT_DTYPE)
            self._copy_stream = torch.cuda.Stream(device=self.device)

    @property
    def h2d_bytes(self) -> int:
        return int(sum(h.numel() * h.element_size() for _, h in self._pairs_in))

    @property
    def d2h_bytes(self) -> int:
        return int(sum(h.numel() * h.element_size() for _, h in self._pairs_out))

    def run_from_host(self, stream=None) -> None:
        import time

        import torch

        if self.streamed:
            self._rec_view["final_now_ns"] = np.iinfo(np.int64).min  # "not finished" marks
        for d, h in self._pairs_in:
            d.copy_(h, non_blocking=True)
        self.run(stream)
        if self.zero_copy:
            return
        if not self.streamed:
            for d, h in self._pairs_out:
                h.copy_(d, non_blocking=True)
            return
        # streamed copy-back: copy each finished prefix of configs (pull order = stamp order)
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        cs = self._copy_stream  # no wait on `main`: that would hold every copy until the kernel ends;
        # a region is copied only after the host saw its configs' fenced records
        fin = self._rec_view["final_now_ns"]
        unset = np.iinfo(np.int64).min
        rb = self.req_base
        (d1, h1), (d2, h2) = self._pairs_out[1], self._pairs_out[2]
        n, done, copied = self.n_cfg, 0, 0
        with torch.cuda.stream(cs):
            while copied < n:
                hi = min(n, done + 8192)
                miss = np.flatnonzero(fin[done:hi] == unset)
                done = done + int(miss[0]) if miss.size else hi
                if done - copied >= self.STREAM_CHUNK_CONFIGS or done == n:
                    lo_r, hi_r = int(rb[copied]), int(rb[done])
                    if hi_r > lo_r:
                        h1[lo_r:hi_r].copy_(d1[lo_r:hi_r], non_blocking=True)
                        h2[lo_r:hi_r].copy_(d2[lo_r:hi_r], non_blocking=True)
                    copied = done
                elif miss.size:
                    time.sleep(2e-4)
        main.wait_stream(cs)

    def host_results(self) -> np.ndarray:
        """The records, in the caller's config order."""
        raw = self._pairs_out[0][1].numpy().view(np.uint8)[: self.n_cfg * SIM_RESULT_DTYPE.itemsize]
        recs = raw.view(SIM_RESULT_DTYPE).copy()
        if self.perm is None:
            return recs
        out = np.empty_like(recs)
        out[self.perm] = recs
        return out

    def host_stamps(self):
        """(first_ns, finish_ns) from pinned host memory, laid out as for the caller's config
        order (config c's requests at [base[c], base[c+1]), base by cumulative sizes)."""
        first, finish = self._pairs_out[1][1].numpy(), self._pairs_out[2][1].numpy()
        n_req = int(self.req_base[-1])
        if self.perm is None:
            return first[:n_req].copy(), finish[:n_req].copy()
        inv = np.empty(self.n_cfg, np.int64)
        inv[self.perm] = np.arange(self.n_cfg)
        sizes = np.diff(self.req_base)[inv]  # caller order
        base = np.zeros(self.n_cfg + 1, np.int64)
        np.cumsum(sizes, out=base[1:])
        cfg_of = np.repeat(np.arange(self.n_cfg), sizes)
        src = self.req_base[:-1][inv][cfg_of] + (np.arange(n_req, dtype=np.int64) - base[:-1][cfg_of])
        return first[src], finish[src]
