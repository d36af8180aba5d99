"""timewarp-b200: the Revati/timewarp hot path (arXiv 2601.00397) on NVIDIA B200.

Batch-duration prediction, Timekeeper min-advance and the discrete-event serving
loop, evaluated in bulk over thousands of emulated configurations by hand-written
sm_100a kernels (libtwb200, include/twb200.h). The Python modules mirror the
reference plugin surface:

  predictor   ConstantPredictor / LinearPredictor / TablePredictor / build_predictor
  timekeeper  BarrierCore op-stream replay and bulk min-advance
  sweep       simulate (drop-in for timewarp.oracle.simulate), simulate_many
  workload    generate_arrivals and CSR packing of workloads
  presets     the BASELINE.json configurations (Llama-3 8B/70B sweeps)
  distributed config sharding across GPUs + NCCL gather of result records
"""

from . import _lib  # noqa: F401

__all__ = ["predictor", "timekeeper", "sweep", "workload", "presets", "distributed", "calibration"]
