"""The BASELINE.json configurations as ready-to-run sweeps.

  config 1  Llama-3-8B TP=1, 1k Poisson requests (qps 8, seed 1)
  config 2  Llama-3-8B TP=4: dispatcher + 4 workers through the Timekeeper, same trace
  config 3  Llama-3-70B TP=4 PP=2, 10k requests (qps 4), prefill/decode mix
  config 4  1,024-config sweep: max_batch_tokens x chunk x max_running x (TP, PP) x policy, 8B
  config 5  65,536 configs: the config-4 grid x {8B, 70B} x 32 workload seeds

Engine defaults for every preset: kv_block_tokens 16, kv_capacity_blocks 32768,
Timekeeper actor grid on with the reference's default 500 us cooldown
(timekeeper.py:36). Models and TP/PP select calibration tables (calibration.py).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import calibration
from .predictor import PredictorSet, TablePredictor
from .sweep import DEFAULT_COOLDOWN_NS, EngineConfig, SchedulingPolicy, SweepConfig, config_array
from .workload import PackedWorkloads, WorkloadSpec, pack_arrays, poisson_arrays

MBT = (1024, 2048, 4096, 8192)
CHUNK = (128, 256, 512, 1024)
MAX_RUNNING = (32, 64, 128, 256)
POLICIES = (SchedulingPolicy.MIXED, SchedulingPolicy.PREFILL_PRIORITIZED)
KV_BLOCK, KV_CAPACITY = 16, 32768


def workload_doc(seed: int = 1, n: int = 1000, qps: float = 8.0) -> dict:
    return {
        "source": "poisson", "qps": qps, "seed": seed, "num_requests": n,
        "prompt_tokens": {"kind": "uniform", "low": 64, "high": 2048},
        "output_tokens": {"kind": "uniform", "low": 16, "high": 256},
    }


def table_index(model: str, tp: int, pp: int) -> int:
    return calibration.MODELS.index(model) * len(calibration.TP_PP_GRID) + calibration.TP_PP_GRID.index((tp, pp))


_PSET = None


def calibration_set() -> PredictorSet:
    """All 16 (model, TP, PP) tables in one blob, ordered as table_index()."""
    global _PSET
    if _PSET is None:
        preds = [
            TablePredictor.from_csv(calibration.csv_path(m, tp, pp), allow_extrapolation=True)
            for m in calibration.MODELS
            for tp, pp in calibration.TP_PP_GRID
        ]
        _PSET = PredictorSet(preds)
    return _PSET


@dataclass
class Sweep:
    name: str
    pset: PredictorSet
    workloads: PackedWorkloads
    configs: list  # SweepConfig
    cfgs: np.ndarray  # SIM_CFG_DTYPE

    def __len__(self) -> int:
        return len(self.configs)

    def subset(self, ids: Sequence[int], name: str | None = None) -> "Sweep":
        ids = np.asarray(ids, np.int64)
        return Sweep(name or f"{self.name}[{len(ids)}]", self.pset, self.workloads,
                     [self.configs[i] for i in ids], self.cfgs[ids].copy())


def _workloads(docs: Sequence[dict]) -> PackedWorkloads:
    return pack_arrays([poisson_arrays(WorkloadSpec.from_doc(d)) for d in docs])


def grid_configs(model: str, workload_id: int, timekeeper: bool = True, cooldown_ns: int = DEFAULT_COOLDOWN_NS):
    out = []
    for mbt, ch, mr, (tp, pp), pol in itertools.product(MBT, CHUNK, MAX_RUNNING, calibration.TP_PP_GRID, POLICIES):
        eng = EngineConfig(chunk_size=ch, policy=pol, max_batch_tokens=mbt, max_running=mr, kv_block_tokens=KV_BLOCK,
                           kv_capacity_blocks=KV_CAPACITY, workers_per_replica=tp, pp_stages=pp)
        out.append(SweepConfig(engine=eng, pred_id=table_index(model, tp, pp), workload_id=workload_id,
                               timekeeper=timekeeper, tk_cooldown_ns=cooldown_ns,
                               label={"model": model, "mbt": mbt, "chunk": ch, "max_running": mr, "tp": tp, "pp": pp,
                                      "policy": pol.value}))
    return out


def sweep_1024(model: str = "8b", seed: int = 1, n_requests: int = 1000, timekeeper: bool = True) -> Sweep:
    """BASELINE config 4 (one workload, 1,024 engine configs)."""
    wl = _workloads([workload_doc(seed, n_requests)])
    cfgs = grid_configs(model, 0, timekeeper)
    return Sweep(f"sweep1024_{model}_seed{seed}", calibration_set(), wl, cfgs, config_array(cfgs))


def sweep_65536(seeds: Sequence[int] = tuple(range(1, 33)), models: Sequence[str] = calibration.MODELS,
                timekeeper: bool = True) -> Sweep:
    """BASELINE config 5: grid x models x workload seeds (65,536 configs by default)."""
    wl = _workloads([workload_doc(s) for s in seeds])
    cfgs = []
    for m in models:
        for w, _ in enumerate(seeds):
            cfgs.extend(grid_configs(m, w, timekeeper))
    return Sweep(f"sweep{len(cfgs)}", calibration_set(), wl, cfgs, config_array(cfgs))


def single(name: str, model: str, tp: int, pp: int, n: int, qps: float, seed: int = 1, timekeeper: bool = True) -> Sweep:
    wl = _workloads([workload_doc(seed, n, qps)])
    eng = EngineConfig(chunk_size=512, max_batch_tokens=2048, max_running=256, kv_block_tokens=KV_BLOCK,
                       kv_capacity_blocks=KV_CAPACITY, workers_per_replica=tp, pp_stages=pp)
    cfg = [SweepConfig(engine=eng, pred_id=table_index(model, tp, pp), workload_id=0, timekeeper=timekeeper,
                       label={"model": model, "tp": tp, "pp": pp})]
    return Sweep(name, calibration_set(), wl, cfg, config_array(cfg))


def config1() -> Sweep:
    return single("config1_8b_tp1", "8b", 1, 1, 1000, 8)


def config2() -> Sweep:
    return single("config2_8b_tp4", "8b", 4, 1, 1000, 8)


def config3() -> Sweep:
    return single("config3_70b_tp4pp2", "70b", 4, 2, 10000, 4)
