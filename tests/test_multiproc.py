"""CPU, world_size 2 and 3 over gloo: the N>1 sweep plumbing.
Every rank holds the same global problem list and takes its LPT share;
the shards are disjoint and cover every problem; each rank's output region
(real placements, produced here by the C restatement, laid out as a plan's
device region) reaches rank 0 by point-to-point sends and decodes to
exactly the placements the owning rank produced; timing takes the max over
ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_08695_b200 import sweep
from paper_2301_08695_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small_sweep():
    graphs, jobs = sweep.global_sweep(graphs=6, vmin=40, vmax=90)
    return graphs, jobs


def _place_all(graphs, jobs, ids):
    """The owning rank's results for problems `ids` (oracle placements)."""
    from oracle import OracleError, Restate
    out = []
    for i in ids:
        gi, n, cap = jobs[i]
        m = W.as_meta_dict(graphs[gi])
        try:
            o = Restate.place(m, 1, [cap] * n, W.COMM_TEST)
            out.append(dict(status=0, device_of=o.device_of, start_us=o.start_us, exec_order=o.exec_order,
                            exec_off=o.exec_off, stats=np.asarray(o.stats, np.int64)))
        except OracleError as e:
            V = m["V"]
            out.append(dict(status=e.kind, device_of=np.full(V, -1, np.int32), start_us=np.zeros(V, np.int64),
                            exec_order=np.zeros(V, np.int32), exec_off=np.zeros(n + 1, np.int32),
                            stats=np.zeros(3, np.int64)))
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    graphs, jobs = _small_sweep()
    ids, sgraphs, sjobs = sweep.rank_shard(rank, world, graphs, jobs)
    mine = _place_all(graphs, jobs, ids)
    region, offs = sweep.pack_region(mine)
    table = np.zeros((len(ids), sweep.OUT_COLS), np.int64)
    table[:, 0] = ids
    table[:, 1:] = offs
    got = sweep.gather_to_root(torch.from_numpy(region), table, dist, torch.device("cpu"))
    t = sweep.max_over_ranks(float(rank + 1), dist, torch.device("cpu"))
    if rank == 0:
        res = sweep.collect(got, lambda i: (graphs[jobs[i][0]]["V"], jobs[i][1]))
        q.put(({i: {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in r.items()} for i, r in res.items()},
               t, [len(g[1]) for g in got]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sweep_gather_moves_real_placements(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, t, per_rank = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == float(world)
    graphs, jobs = _small_sweep()
    P = len(jobs)
    assert sorted(res) == list(range(P)) and sum(per_rank) == P and all(c > 0 for c in per_rank)
    want = _place_all(graphs, jobs, range(P))  # every problem placed locally
    for i in range(P):
        for k in ("status", "device_of", "start_us", "exec_order", "exec_off", "stats"):
            assert np.array_equal(np.asarray(res[i][k]), np.asarray(want[i][k])), (i, k)


def test_lpt_partition_balanced_and_deterministic():
    costs = [10, 9, 8, 7, 6, 5, 4, 3, 2, 1]
    parts = sweep.lpt_partition(costs, 3)
    assert sorted(sum(parts, [])) == list(range(10))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= 2
    assert parts == sweep.lpt_partition(costs, 3)


def test_shards_cover_the_sweep_at_every_world_size():
    graphs, jobs = sweep.global_sweep(graphs=64)
    P = len(jobs)
    assert P == 4096
    costs = sweep.problem_costs(graphs, jobs)
    for world in (1, 2, 4, 8):
        seen = []
        loads = []
        for r in range(world):
            ids, sg, sj = sweep.rank_shard(r, world, graphs, jobs)
            seen += ids
            loads.append(sum(costs[i] for i in ids))
            for k, i in enumerate(ids):  # remapped jobs point at the same graph and roster
                assert sg[sj[k][0]] is graphs[jobs[i][0]] and sj[k][1:] == jobs[i][1:]
        assert sorted(seen) == list(range(P))
        assert max(loads) / (sum(loads) / world) < 1.01  # LPT over 4096 problems is nearly even


def test_pack_and_decode_roundtrip():
    graphs, jobs = _small_sweep()
    res = _place_all(graphs, jobs, range(5))
    region, offs = sweep.pack_region(res)
    for i, r in enumerate(res):
        row = np.concatenate([[i], offs[i]])
        V, n = graphs[jobs[i][0]]["V"], jobs[i][1]
        d = sweep.decode(region, row, V, n)
        for k in ("device_of", "start_us", "exec_order", "exec_off", "stats"):
            assert np.array_equal(d[k], r[k])
        assert d["status"] == r["status"]
