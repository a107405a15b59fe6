"""Multi-GPU batched sweep: the reference's OpenMP fan-out
over problems (proj/src/bench.cpp:105-237, ``#pragma omp parallel for`` at
:121) becomes one process per GPU.

* The SAME global problem list on every rank (the C5 sweep: 64 graphs x
  {2,4,8,16} devices x 16 caps = 4096 problems), split by a deterministic
  longest-processing-time partition on the estimated cost V*n (ties by
  problem id): strong scaling, total work fixed.
* Each rank places its shard on its own GPU; no inter-GPU traffic while
  placing.
* One collective at the end: every rank's device-resident output region
  (device_of, start_us, exec_order, exec_off, stats and status of each of
  its problems, exactly the bytes bx_plan_download copies) goes to rank 0
  over NCCL point-to-point (NCCL has no variable-size gather), with the
  per-problem offsets into it; rank 0 decodes the full results ordered by
  problem id.
"""
from __future__ import annotations

import numpy as np

OUT_COLS = 7  # problem id, then byte offsets of device_of, start, exec_order, exec_off, stats, status record


def global_sweep(graphs: int = 64, vmin: int = 1000, vmax: int = 20000):
    """The sweep every rank agrees on: (graph dicts, jobs [(graph, n, cap)])."""
    from . import workloads as W
    gs = W.sweep_graphs(0, graphs, vmin, vmax)
    return gs, W.sweep_jobs(gs)


def lpt_partition(costs, world: int):
    """Deterministic longest-processing-time partition of problem ids over
    `world` ranks: problems by descending cost (ties by id) each go to the
    least-loaded rank (ties by rank). Returns per-rank ascending id lists."""
    import heapq
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(world)]
    parts = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(p) for p in parts]


def problem_costs(graphs, jobs):
    return [graphs[g]["V"] * n for g, n, _ in jobs]


def rank_shard(rank: int, world: int, graphs, jobs):
    """Rank `rank`'s problems: (global ids, the graphs they use, jobs with
    graph indices remapped into that list)."""
    ids = lpt_partition(problem_costs(graphs, jobs), world)[rank]
    used = sorted({jobs[i][0] for i in ids})
    remap = {g: k for k, g in enumerate(used)}
    return ids, [graphs[g] for g in used], [(remap[jobs[i][0]], jobs[i][1], jobs[i][2]) for i in ids]


class _DeviceBytes:
    """A raw device range as a zero-copy uint8 tensor (CUDA array interface)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def region_tensor(plan, device):
    """The plan's device-resident output region as a uint8 torch tensor view."""
    import torch
    ptr, nbytes = plan.output_region()
    if nbytes == 0:
        return torch.zeros(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_DeviceBytes(ptr, nbytes), device=device)


def offsets_table(plan, ids):
    """[P, OUT_COLS] int64: global id + the six byte offsets of each job."""
    t = np.zeros((len(ids), OUT_COLS), np.int64)
    for k, i in enumerate(ids):
        t[k, 0] = i
        t[k, 1:] = plan.job_outputs(k)
    return t


def gather_to_root(region, table: np.ndarray, dist, device=None):
    """Rank 0 receives every rank's (output region, offsets table) over
    point-to-point sends (NCCL on the GPU box, gloo in the CPU tests).
    Returns [(region uint8 numpy, table)] per rank on rank 0, None elsewhere."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = device if device is not None else region.device
    sizes = torch.tensor([region.numel(), table.shape[0]], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    tab = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
    if rank != 0:
        ops = [dist.P2POp(dist.isend, region.to(dev), 0), dist.P2POp(dist.isend, tab, 0)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        return None
    bufs = [(region.to(dev), tab)]
    ops = []
    for r in range(1, world):
        nb, npr = (int(x) for x in all_sizes[r].tolist())
        rb = torch.empty(nb, dtype=torch.uint8, device=dev)
        rt = torch.empty((npr, OUT_COLS), dtype=torch.int64, device=dev)
        ops += [dist.P2POp(dist.irecv, rb, r), dist.P2POp(dist.irecv, rt, r)]
        bufs.append((rb, rt))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return [(b.cpu().numpy(), t.cpu().numpy()) for b, t in bufs]


def decode(region: np.ndarray, row: np.ndarray, V: int, n: int) -> dict:
    """One problem's outputs out of a gathered region (bx_plan_job_outputs)."""
    def arr(off, dt, count):
        return np.frombuffer(region, dtype=dt, count=count, offset=int(off))

    status = int(arr(row[6], np.int32, 1)[0])
    return dict(id=int(row[0]), status=status, device_of=arr(row[1], np.int32, V), start_us=arr(row[2], np.int64, V),
                exec_order=arr(row[3], np.int32, V), exec_off=arr(row[4], np.int32, n + 1),
                stats=arr(row[5], np.int64, 3))


def collect(gathered, sizes_of):
    """Rank 0: {global id: decoded result} from gather_to_root's output;
    sizes_of(id) -> (V, n)."""
    out = {}
    for region, table in gathered:
        for row in table:
            V, n = sizes_of(int(row[0]))
            out[int(row[0])] = decode(region, row, V, n)
    return out


def pack_region(results):
    """Test helper: lays out results [{device_of, start_us, exec_order,
    exec_off, stats, status}] the way a plan's output region does (8-byte
    aligned arrays per job) and returns (region uint8, offsets [P, 6])."""
    chunks, offs, pos = [], [], 0

    def put(a):
        nonlocal pos
        pos = (pos + 7) & ~7
        at = pos
        b = np.ascontiguousarray(a).tobytes()
        chunks.append((at, b))
        pos += max(len(b), 1)
        return at

    for r in results:
        o = [0] * 6
        o[4] = put(np.asarray(r["stats"], np.int64))
        o[5] = put(np.array([r["status"], 0, 0, 0, 0, 0, 0, 0, 0, 0], np.int32))
        o[1] = put(np.asarray(r["start_us"], np.int64))
        o[0] = put(np.asarray(r["device_of"], np.int32))
        o[2] = put(np.asarray(r["exec_order"], np.int32))
        o[3] = put(np.asarray(r["exec_off"], np.int32))
        offs.append(o)
    region = np.zeros(pos, np.uint8)
    for at, b in chunks:
        region[at:at + len(b)] = np.frombuffer(b, np.uint8)
    return region, np.array(offs, np.int64).reshape(-1, 6)


def max_over_ranks(x: float, dist, device=None) -> float:
    """Timing rule: the job time is the slowest rank's."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
