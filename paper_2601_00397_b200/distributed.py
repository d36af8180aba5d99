"""Multi-GPU sweeps: independent configs sharded across ranks, results merged with NCCL.

Configs share nothing during emulation (each config's Timekeeper min is over its
own actors), so the data path has no collective at all. Each rank
runs its shard with one persistent tw_sim_many launch; the only collective is a
single all-gather of the fixed-size 64-byte result records (plus their config
ids) at the end, over NCCL/NVLink (gloo on CPU for tests), after which every rank
holds the merged table ordered by config id.
"""

from __future__ import annotations

import heapq

import numpy as np

from ._lib import SIM_RESULT_DTYPE


def partition(costs: np.ndarray, world: int) -> list:
    """Greedy longest-processing-time partition of config ids over `world` ranks.

    Deterministic (stable tie-breaks), so every rank computes the same plan with no
    communication.
    """
    costs = np.asarray(costs, np.float64)
    order = np.argsort(-costs, kind="stable")
    heap = [(0.0, r) for r in range(world)]
    shards: list = [[] for _ in range(world)]
    for c in order:
        load, r = heapq.heappop(heap)
        shards[r].append(int(c))
        heapq.heappush(heap, (load + float(costs[c]), r))
    return [np.sort(np.asarray(s, np.int64)) for s in shards]


def records_to_tensor(ids: np.ndarray, results: np.ndarray, max_local: int, device):
    """Pack (config id, 64-byte record) rows into an int64 [max_local, 9] tensor (id -1 = padding)."""
    import torch

    rows = np.full((max_local, 9), -1, np.int64)
    n = len(ids)
    rows[:n, 0] = ids
    rows[:n, 1:] = np.ascontiguousarray(results).view(np.int64).reshape(n, 8)
    return torch.from_numpy(rows).to(device)


def gather_records_device(ids_dev, records, n_total: int, max_local: int, device, group=None):
    """The sweep's merge step, device-resident: all-gather every rank's (config id, 64-byte
    record) rows with one collective (NCCL over NVLink between GPUs), then scatter them
    into an [n_total, 8] int64 table ordered by config id on `device`. `records` is the
    rank's raw record bytes (a device tensor, or pinned host memory when the kernel wrote
    them zero-copy); stream-ordered, no host synchronisation. Returns (merged, rows)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = ids_dev.numel()
    local = torch.full((max_local, 9), -1, dtype=torch.int64, device=device)
    local[:n, 0] = ids_dev
    rec = records[: n * SIM_RESULT_DTYPE.itemsize].view(torch.int64).view(n, 8)
    local[:n, 1:].copy_(rec, non_blocking=True)
    rows = torch.empty((world * max_local, 9), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(rows, local, group=group)
    # padding rows (id -1) land in a spare row n_total: no host sync for a boolean mask
    idx = torch.where(rows[:, 0] >= 0, rows[:, 0], torch.full_like(rows[:, 0], n_total))
    merged = torch.zeros((n_total + 1, 8), dtype=torch.int64, device=device)
    merged.index_copy_(0, idx, rows[:, 1:])
    return merged[:n_total], rows


def gather_results(ids: np.ndarray, results: np.ndarray, n_total: int, max_local: int, device, group=None) -> np.ndarray:
    """All-gather every rank's records; returns the merged SIM_RESULT_DTYPE[n_total] on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    local = records_to_tensor(ids, results, max_local, device)
    outs = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(outs, local, group=group)  # NCCL over NVLink; gloo in the CPU tests
    rows = torch.cat(outs).cpu().numpy()
    rows = rows[rows[:, 0] >= 0]
    merged = np.zeros(n_total, SIM_RESULT_DTYPE)
    merged_i64 = merged.view(np.int64).reshape(n_total, 8)
    merged_i64[rows[:, 0]] = rows[:, 1:]
    if len(np.unique(rows[:, 0])) != n_total:
        raise RuntimeError("config ids missing or duplicated after the gather")
    return merged
