"""Multi-GPU batched sweep plumbing.

Independent placement problems shard across ranks with no inter-GPU
traffic; the only collective is the final gather of per-problem summaries
(NCCL over NVLink on the GPU box; gloo in the CPU tests). One process per
GPU, launched by torchrun.
"""
from __future__ import annotations

import numpy as np

SUMMARY_COLS = 4  # status, checksum(start*131 + device), makespan estimate, problem id


def rank_sweep(rank: int, graphs_per_rank: int = 64, vmin: int = 1000, vmax: int = 20000):
    """Rank r's shard: its own 64-graph sweep (graph seeds offset by r), so
    per-GPU work is fixed as the GPU count grows (weak scaling)."""
    from . import workloads as W
    graphs = W.sweep_graphs(rank, graphs_per_rank, vmin, vmax)
    return graphs, W.sweep_jobs(graphs)


def lpt_partition(costs, world: int):
    """Deterministic longest-processing-time partition of problem ids over
    `world` ranks (ties by id): used when one global problem list is split
    instead of generated per rank."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0] * world
    parts = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda x: (load[x], x))
        parts[r].append(i)
        load[r] += costs[i]
    return [sorted(p) for p in parts]


def summarize(statuses, placements, k_of, base_id: int = 0):
    """Per-problem summary rows: (status, checksum, finish estimate, id)."""
    P = len(statuses)
    out = np.zeros((P, SUMMARY_COLS), np.int64)
    for i in range(P):
        out[i, 0] = statuses[i]
        out[i, 3] = base_id + i
        p = placements[i]
        if statuses[i] == 0 and p is not None and len(p.start_us):
            out[i, 1] = int((p.start_us * 131 + p.device_of).sum())
            out[i, 2] = int((p.start_us + k_of(i)).max())
    return out


def gather_summaries(summary: np.ndarray, dist, device=None):
    """All-gather every rank's summary rows (the sweep's one collective).
    Returns the concatenated [world*P, cols] array ordered by rank."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(summary))
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return torch.cat(parts, 0).cpu().numpy()


def max_over_ranks(x: float, dist, device=None) -> float:
    """Timing rule: the job time is the slowest rank's."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
