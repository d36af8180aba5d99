#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (run in the build container).

    python scripts/ncu_summary.py gpurun_out/prof_sim.ncu-rep > profiles/r01_k_sim.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/r01_launches.md
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize_report(path):
    rows = ncu_csv(["-i", path, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: `{path}`\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## kernel `{d.get('Kernel Name', '?')}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        print()
    # stall reasons from the SASS source page
    src = ncu_csv(["-i", path, "--page", "source", "--csv", "--print-source=sass"])
    if len(src) > 2:
        hdr = src[1]
        idx = {h: i for i, h in enumerate(hdr)}
        data = src[2:]
        reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data) or 1
        agg = {h: sum(int(r[idx[h]] or 0) for r in data) for h in reasons}
        print("## warp stall sampling (share of all samples)\n")
        print("| reason | share |\n|---|---|")
        for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
            print(f"| {k} | {100 * v / tot:.1f}% |")
        ops = collections.Counter()
        for r in data:
            s = r[1].strip().split()
            if not s:
                continue
            op = s[1] if s[0].startswith("@") and len(s) > 1 else s[0]
            ops[op.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
        total = sum(ops.values()) or 1
        print("\n## executed SASS opcode mix (warp-level)\n")
        print("| opcode | share |\n|---|---|")
        for k, v in ops.most_common(14):
            print(f"| {k} | {100 * v / total:.1f}% |")
        print(f"\ntotal warp instructions executed: {total}")


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1 :]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "second": 1e6, "s": 1e6}[unit]
        agg[name][0] += 1
        agg[name][1] += v * scale
    total = sum(v[1] for v in agg.values()) or 1
    print(f"# ncu launch list: `{path}` (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:90]}` | {n} | {t:.1f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarize_launches(sys.argv[2])
    else:
        summarize_report(sys.argv[1])
