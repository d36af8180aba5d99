"""Synthetic calibration tables for the Llama-3-8B / 70B sweep presets.

The reference ships no model calibrations (parity-unpinned
north-star features), so models and TP/PP degrees are expressed as *which table a
config uses*, which keeps every prediction inside the reference's TablePredictor
semantics. The tables follow SURVEY.md §8d:

    11 x 11 grid, P in {0, 16, 32, ..., 8192}, D in {0, 1, 2, 4, ..., 512} minus (0, 0)
    us = floor(s * (800 + 9 P + 35 D + 0.002 P D))
    8B:  s = (1 + 0.1 (PP - 1)) / sqrt(TP)
    70B: s = 8 sqrt(2) (1 + 0.1 (PP - 1)) / sqrt(TP)

They are written as CSV files so the reference's TablePredictor.from_csv and this
engine read byte-identical rows (frozen copies live in calib/).
"""

from __future__ import annotations

import math
import os

PREFILL_AXIS = (0, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192)
DECODE_AXIS = (0, 1, 2, 4, 8, 16, 32, 64, 128, 256, 512)
MODELS = ("8b", "70b")
TP_PP_GRID = ((1, 1), (2, 1), (4, 1), (8, 1), (1, 2), (2, 2), (4, 2), (8, 2))

CALIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "calib")


def scale(model: str, tp: int, pp: int) -> float:
    base = (1.0 + 0.1 * (pp - 1)) / math.sqrt(tp)
    if model == "8b":
        return base
    if model == "70b":
        return 8.0 * math.sqrt(2.0) * base
    raise ValueError(f"unknown model preset {model!r}")


def table_rows(model: str, tp: int, pp: int) -> dict:
    s = scale(model, tp, pp)
    rows = {}
    for p in PREFILL_AXIS:
        for d in DECODE_AXIS:
            if p == 0 and d == 0:
                continue
            rows[(p, d)] = int(math.floor(s * (800 + 9 * p + 35 * d + 0.002 * p * d)))
    return rows


def csv_path(model: str, tp: int, pp: int, directory: str | None = None) -> str:
    return os.path.join(directory or CALIB_DIR, f"llama3_{model}_tp{tp}_pp{pp}.csv")


def write_csvs(directory: str | None = None) -> list[str]:
    directory = directory or CALIB_DIR
    os.makedirs(directory, exist_ok=True)
    paths = []
    for m in MODELS:
        for tp, pp in TP_PP_GRID:
            path = csv_path(m, tp, pp, directory)
            with open(path, "w", newline="") as fh:
                fh.write("total_prefill_tokens,num_decodes,duration_us\n")
                for (p, d), us in sorted(table_rows(m, tp, pp).items()):
                    fh.write(f"{p},{d},{us}\n")
            paths.append(path)
    return paths


if __name__ == "__main__":  # regenerate the frozen copies
    for p in write_csvs():
        print(p)
