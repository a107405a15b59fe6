"""GPU parity for the simulators on hand-made placements: random device
assignments and FIFO orders (valid topological ones and deadlocking ones),
ample / tight / permanent-memory-violating capacities, both memory modes and
both comm modes, with and without zero-duration nodes. Parallel comm mode
without zero-duration nodes runs the dataflow kernel (K4f), sequential comm
mode on <= 32 devices its transfer sequencer, everything else the event-loop
kernel (K4); all must match the C restatement of simulator.cpp bit for bit,
error texts included."""
import heapq

import numpy as np
import pytest

from oracle import OracleError, Restate
from paper_2301_08695_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _topo(m, rng):
    V = m["V"]
    indeg = np.zeros(V, np.int64)
    np.add.at(indeg, m["edst"], 1)
    out = [[] for _ in range(V)]
    for s, d in zip(m["esrc"].tolist(), m["edst"].tolist()):
        out[s].append(d)
    pri = rng.random(V)
    h = [(pri[j], j) for j in range(V) if indeg[j] == 0]
    heapq.heapify(h)
    order = []
    while h:
        _, j = heapq.heappop(h)
        order.append(j)
        for c in out[j]:
            indeg[c] -= 1
            if indeg[c] == 0:
                heapq.heappush(h, (pri[c], c))
    return order


def _placement(bx, m, n, rng, deadlock=False):
    V = m["V"]
    dev = rng.integers(0, n, V).astype(np.int32)
    order = _topo(m, rng)
    lists = [[j for j in order if dev[j] == d] for d in range(n)]
    if deadlock:
        d = int(np.argmax([len(x) for x in lists]))
        lists[d] = lists[d][::-1]
    flat = np.array([j for x in lists for j in x], np.int32)
    off = np.cumsum([0] + [len(x) for x in lists]).astype(np.int32)
    return bx.Placement("manual", dev, np.zeros(V, np.int64), flat, off)


def _graphs():
    out = []
    for seed in range(3):
        out += [W.layered_dag(6, 10, seed), W.grid_chain(15, 5, seed), W.branchy(5, seed),
                W.wide_random(120, seed)]
    return out


def _check(bx, m, gg, pl, caps, cm, mm, options=None):
    try:
        o = Restate.simulate(m, caps, cm, mm, pl.device_of, pl.exec_order_flat, pl.exec_off)
        oe = None
    except OracleError as e:
        oe = (e.kind, e.msg)
    try:
        r = bx.simulate(gg, pl, caps, bx.CommModel(*cm), mm, options=options)
        re = None
    except bx.Error as e:
        re = (e.kind, e.msg)
    assert oe == re
    if oe is None:
        assert r.makespan_us == o.makespan
        assert np.array_equal(r.start_us, o.start_us)
        assert r.peak_bytes.tolist() == o.peak.tolist()
        assert r.busy_us.tolist() == o.busy.tolist()
        assert r.idle_us.tolist() == o.idle.tolist()
        assert [r.transfer_count, r.transfer_bytes, r.duplicate_transfers, r.cache_hits] == [
            o.transfer_count, o.transfer_bytes, o.duplicate_transfers, o.cache_hits]
    return oe


@pytest.mark.parametrize("gi", range(12))
def test_sim_random_placements(bx, gi):
    g = _graphs()[gi]
    rng = np.random.default_rng(100 + gi)
    seen_err = set()
    for zero in (False, True):
        m = W.as_meta_dict(g)
        if zero:
            k = m["k"].copy()
            k[rng.random(len(k)) < 0.3] = 0
            m = dict(m, k=k)
        gg = bx.MetaGraph.from_dict(m)
        need = m["perm"] + m["out"] + m["temp"]
        for n in (1, 2, 3, 5, 8):
            for trial in range(3):
                pl = _placement(bx, m, n, rng, deadlock=(trial == 2 and n > 1))
                perm_d = np.bincount(pl.device_of, weights=m["perm"], minlength=n).astype(np.int64)
                tot_d = np.bincount(pl.device_of, weights=need, minlength=n).astype(np.int64)
                for caps in (tot_d + 1, perm_d + (tot_d - perm_d) // 4, np.maximum(perm_d - 1, 0)):
                    caps = [int(c) for c in caps]
                    for cm in ((12.5, 0.002, 1), (0.0, 0.0, 1), (5.0, 0.001, 0)):
                        for mm in (0, 1):
                            oe = _check(bx, m, gg, pl, caps, cm, mm)
                            seen_err.add(None if oe is None else oe[0])
    assert None in seen_err and len(seen_err) >= 2  # both successes and errors were exercised


SEQ = (5.0, 0.001, 0)


@pytest.mark.parametrize("cmt", [W.COMM_TEST, SEQ], ids=["parallel", "sequential"])
def test_sim_flow_full_size_vs_event_loop(bx, cmt):
    """100k-op m-ETF placement: the dataflow kernel (parallel comm) and the
    transfer sequencer (sequential comm) against the C restatement in both
    memory modes (full-size, bit-exact)."""
    g = W.layered_dag_fast(100, 1000, 3)
    m = W.as_meta_dict(g)
    gg = bx.MetaGraph.from_dict(m)
    cm = bx.CommModel(*cmt)
    caps = np.full(4, W.bench_capacity(g, 4, 1.2), np.int64)
    plan = bx.Plan([gg], [bx.Job(0, "m-etf", caps, cm)])
    plan.upload()
    plan.place()
    plan.download()
    p = plan.result(0)
    for mm in (0, 1):
        plan.simulate(mm)
        r = plan.sim_download()[0]
        o = Restate.simulate(m, caps, cmt, mm, p.device_of, p.exec_order_flat, p.exec_off)
        assert r.makespan_us == o.makespan and np.array_equal(r.start_us, o.start_us)
        assert r.peak_bytes.tolist() == o.peak.tolist() and r.idle_us.tolist() == o.idle.tolist()
        assert [r.transfer_count, r.transfer_bytes, r.duplicate_transfers, r.cache_hits] == [
            o.transfer_count, o.transfer_bytes, o.duplicate_transfers, o.cache_hits]
    plan.close()


def test_sim_many_devices_and_tiny_graphs(bx):
    """Walker warps owning several devices (n = 40 > 32 warps), the sequencer
    at its 32-lane limit and the event loop past it (sequential comm, n = 32
    and 40), and degenerate graphs (one node, isolated nodes, empty device
    FIFOs)."""
    rng = np.random.default_rng(5)
    g = W.layered_dag(10, 30, 3)
    m = W.as_meta_dict(g)
    gg = bx.MetaGraph.from_dict(m)
    need = m["perm"] + m["out"] + m["temp"]
    for n, cm in ((40, (12.5, 0.002, 1)), (32, SEQ), (40, SEQ), (32, (0.0, 0.0, 0))):
        for trial in range(4):
            pl = _placement(bx, m, n, rng, deadlock=trial == 3)
            tot_d = np.bincount(pl.device_of, weights=need, minlength=n).astype(np.int64)
            for caps in (tot_d + 1, tot_d // 2 + 1):
                for mm in (0, 1):
                    _check(bx, m, gg, pl, [int(c) for c in caps], cm, mm)
    one = dict(V=1, E=0, k=np.array([7], np.int64), temp=np.array([3], np.int64), perm=np.array([5], np.int64),
               out=np.array([2], np.int64), esrc=np.zeros(0, np.int32), edst=np.zeros(0, np.int32),
               ebytes=np.zeros(0, np.int64))
    iso = dict(V=3, E=0, k=np.array([4, 9, 1], np.int64), temp=np.zeros(3, np.int64), perm=np.ones(3, np.int64),
               out=np.ones(3, np.int64), esrc=np.zeros(0, np.int32), edst=np.zeros(0, np.int32),
               ebytes=np.zeros(0, np.int64))
    for mg, n in ((one, 1), (one, 3), (iso, 2), (iso, 5)):
        gm = bx.MetaGraph.from_dict(mg)
        pl = _placement(bx, mg, n, rng)
        for mm in (0, 1):
            for cm in ((12.5, 0.002, 1), SEQ):
                _check(bx, mg, gm, pl, [100] * n, cm, mm)


@pytest.mark.parametrize("cmt", [W.COMM_TEST, SEQ], ids=["parallel", "sequential"])
def test_sim_batched_plan_vs_restatement(bx, cmt):
    """A many-job plan (> 148 problems: 256-thread walker / sequencer CTAs,
    several devices per warp at n = 16) placed and simulated on the device,
    every report against the C restatement."""
    graphs = W.sweep_graphs(3, 8, 800, 3000)
    jobs = [(gi, n, W.bench_capacity(graphs[gi], n, f)) for gi in range(len(graphs)) for n in (2, 5, 16)
            for f in (1.05, 1.3, 1.6, 2.0, 3.0, 4.0, 5.0)]
    assert len(jobs) > 148
    mgs = [bx.MetaGraph.from_dict(W.as_meta_dict(g)) for g in graphs]
    plan = bx.Plan(mgs, [bx.Job(gi, "m-etf", np.full(n, cap, np.int64), bx.CommModel(*cmt)) for gi, n, cap in jobs])
    plan.upload()
    plan.place()
    plan.download()
    for mm in (0, 1):
        plan.simulate(mm)
        reps = plan.sim_download()
        for i, (gi, n, cap) in enumerate(jobs):
            st, _ = plan.status(i)
            if st:
                continue
            p = plan.result(i)
            m = W.as_meta_dict(graphs[gi])
            try:
                o = Restate.simulate(m, [cap] * n, cmt, mm, p.device_of, p.exec_order_flat, p.exec_off)
            except OracleError as e:
                assert reps[i] == (e.kind, e.msg), i
                continue
            r = reps[i]
            assert not isinstance(r, tuple), (i, r)
            assert r.makespan_us == o.makespan and np.array_equal(r.start_us, o.start_us), i
            assert r.peak_bytes.tolist() == o.peak.tolist(), i
            assert [r.transfer_count, r.transfer_bytes, r.cache_hits] == [o.transfer_count, o.transfer_bytes,
                                                                          o.cache_hits], i
    plan.close()


@pytest.mark.parametrize("cap", ["0", "3"])
def test_event_heap_spill(bx, cap):
    """The event-loop kernel's heap starting in a 3-entry shared-memory slice
    (spills to global memory at once) or in global memory outright: same
    reports and errors, sequential comm and zero-duration nodes."""
    rng = np.random.default_rng(9)
    for g in (W.layered_dag(6, 10, 1), W.branchy(5, 2)):
        m = W.as_meta_dict(g)
        k = m["k"].copy()
        k[rng.random(len(k)) < 0.3] = 0
        for mg in (m, dict(m, k=k)):
            gg = bx.MetaGraph.from_dict(mg)
            need = mg["perm"] + mg["out"] + mg["temp"]
            for n in (2, 5):
                pl = _placement(bx, mg, n, rng)
                tot_d = np.bincount(pl.device_of, weights=need, minlength=n).astype(np.int64)
                for caps in (tot_d + 1, tot_d // 3 + 1):
                    for cm in ((5.0, 0.001, 0), (12.5, 0.002, 1)):
                        for mm in (0, 1):
                            _check(bx, mg, gg, pl, [int(c) for c in caps], cm, mm,
                                   options={"sim_heap_cap": int(cap)})
