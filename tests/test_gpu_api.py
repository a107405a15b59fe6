"""GPU: the placer API beside the entry points, against the reference.

* schedulable_time (placers.hpp:66-67): the test_placers.cpp:52-79 KATs
  (5 / 7 / 8 / 6) and random partial schedules vs the compiled reference;
* critical_path_us (simulator.cpp:296-309) vs the reference, and its
  CycleError;
* SimOptions::record_trace + trace_to_csv (simulator.cpp:60-64, 311-324) vs
  the reference's CSV, both comm modes, both memory modes;
* the one-shot entry points in steady state (arena reuse) and a plan's
  simulate of jobs that never got a placement.
"""
import numpy as np
import pytest

import kats
from oracle import OracleError, Ref, Restate
from paper_2301_08695_b200 import workloads as W

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not Ref.available(), reason="compiled reference (oracle/_ref) missing")


def _sched_kat_graph(bx):
    # Node 2 consumes node 0 (placed) over a 2us edge (test_placers.cpp:53-56)
    g = kats.graph([kats.node(0, 5), kats.node(1, 1), kats.node(2, 3)], [(0, 2, 2)])
    return bx.MetaGraph.from_dict(g)


def test_schedulable_time_kats(bx):
    gg = _sched_kat_graph(bx)
    cm = bx.CommModel(0.0, 1.0, bx.SEQUENTIAL)  # c = bytes

    def fresh():
        st = bx.PlacerState(3, 2, bx.SEQUENTIAL)
        st.device_of[0] = 0
        st.finish_us[0] = 5
        return st

    st = fresh()
    st.dev_free[0] = 3
    assert bx.schedulable_time(st, 2, 0, gg, cm) == 5      # parent on the same device
    st = fresh()
    assert bx.schedulable_time(st, 2, 1, gg, cm) == 7      # remote parent, idle queues
    st = fresh()
    st.xfer_tail[0] = 6
    assert bx.schedulable_time(st, 2, 1, gg, cm) == 8      # behind a busy sender queue
    st = fresh()
    st.cache_arrival[0 * 2 + 1] = 6
    st.xfer_tail[0] = 100
    assert bx.schedulable_time(st, 2, 1, gg, cm) == 6      # cached tensor costs nothing new
    before = st.xfer_tail.copy()
    bx.schedulable_time(st, 2, 1, gg, cm)
    assert np.array_equal(st.xfer_tail, before)             # an estimate never mutates the state


def _random_state(rng, m, n, mode):
    V = m["V"]
    st_dev = np.full(V, -1, np.int32)
    fin = np.zeros(V, np.int64)
    placed = rng.random(V) < 0.6
    st_dev[placed] = rng.integers(0, n, placed.sum())
    fin[placed] = rng.integers(0, 5000, placed.sum())
    cache = np.full(V * n, -1, np.int64)
    hit = rng.random(V * n) < 0.2
    cache[hit] = rng.integers(0, 6000, hit.sum())
    return dict(dev_free=rng.integers(0, 4000, n).astype(np.int64),
                tail=rng.integers(0, 4000, n).astype(np.int64), device_of=st_dev, finish=fin, cache=cache)


@needs_ref
@pytest.mark.parametrize("mode", [0, 1])
def test_schedulable_time_random_states_vs_reference(bx, mode):
    rng = np.random.default_rng(7 + mode)
    for gi, g in enumerate((W.layered_dag(6, 10, 1), W.branchy(4, 2), W.wide_random(120, 3))):
        m = W.as_meta_dict(g)
        rg = Ref.graph(W.as_ref_base(g), pipeline=-1)
        gg = bx.MetaGraph.from_dict(m)
        for n in (1, 3, 8):
            s = _random_state(rng, m, n, mode)
            cmv = (12.5, 0.002, mode)
            st = bx.PlacerState(m["V"], n, mode)
            st.dev_free[:] = s["dev_free"]
            st.xfer_tail[:] = s["tail"]
            st.device_of[:] = s["device_of"]
            st.finish_us[:] = s["finish"]
            st.cache_arrival[:] = s["cache"]
            js, ps, want = [], [], []
            for j in range(m["V"]):
                parents = m["esrc"][m["edst"] == j]
                if mode == 0 and (s["device_of"][parents] < 0).any():
                    continue  # the reference indexes tail(-1) there (undefined)
                for p in range(n):
                    js.append(j)
                    ps.append(p)
                    want.append(Ref.schedulable_time(rg, n, cmv, s["dev_free"], s["tail"], s["device_of"],
                                                     s["finish"], s["cache"], j, p))
            got = bx.schedulable_times(st, js, ps, gg, bx.CommModel(*cmv))
            assert np.array_equal(got, np.array(want, np.int64)), (gi, n)


def test_schedulable_time_errors(bx):
    gg = _sched_kat_graph(bx)
    st = bx.PlacerState(3, 2, bx.SEQUENTIAL)  # node 0 unplaced
    with pytest.raises(bx.ValidationError, match="unplaced"):
        bx.schedulable_time(st, 2, 1, gg, bx.CommModel(0.0, 1.0, bx.SEQUENTIAL))
    with pytest.raises(bx.ValidationError, match="out of range"):
        bx.schedulable_time(st, 3, 0, gg, bx.CommModel())
    st = bx.PlacerState(3, 2, bx.PARALLEL)  # parallel mode: finish + c of an unplaced parent
    assert bx.schedulable_time(st, 2, 1, gg, bx.CommModel(0.0, 1.0, bx.PARALLEL)) == 2


@needs_ref
def test_critical_path_vs_reference(bx):
    for g in (W.layered_dag(20, 30, 4), W.branchy(10, 5), W.grid_chain(40, 5, 6), W.wide_random(2000, 7),
              W.layered_dag_fast(200, 500, 8)):
        m = W.as_meta_dict(g)
        rg = Ref.graph(W.as_ref_base(g), pipeline=-1)
        assert bx.critical_path_us(bx.MetaGraph.from_dict(m)) == Ref.critical_path(rg)
    assert bx.critical_path_us(bx.MetaGraph.from_dict(kats.chain(4, k=5))) == 20
    assert bx.critical_path_us(bx.MetaGraph([], [], [], [], [], [], [])) == 0


def test_critical_path_cycle_error(bx):
    # a meta graph with a cycle (the transforms never produce one; raw input can)
    gg = bx.MetaGraph([1, 2, 3], [0] * 3, [0] * 3, [0] * 3, [0, 1, 2], [1, 2, 1], [0, 0, 0], first_id=[10, 11, 12])
    with pytest.raises(bx.CycleError, match=r"groups of base node ids \{11, 12\} remain"):
        bx.critical_path_us(gg)


@needs_ref
@pytest.mark.parametrize("mode", [0, 1])
def test_trace_csv_vs_reference(bx, mode):
    rng = np.random.default_rng(11 + mode)
    for gi, g in enumerate((W.branchy(5, 3), W.layered_dag(8, 12, 4), W.wide_random(300, 5))):
        m = W.as_meta_dict(g)
        rg = Ref.graph(W.as_ref_base(g), pipeline=-1)
        gg = bx.MetaGraph.from_dict(m)
        for n in (2, 5):
            caps = [W.bench_capacity(g, n, 1.5)] * n
            cmv = (12.5, 0.002, mode)
            for algo in ("m-etf", "random"):
                if algo == "m-etf":
                    o = Restate.place(m, 1, caps, cmv)
                    dev, eo, off = o.device_of, o.exec_order, o.exec_off
                else:  # a random valid placement: topological FIFO order per device
                    dev = rng.integers(0, n, m["V"]).astype(np.int32)
                    dev, eo, off = kats.manual(dev, n)
                for mem in (0, 1):
                    try:
                        rtext, rcount = Ref.simulate_trace_csv(rg, caps, cmv, mem, dev, eo, off)
                        rerr = None
                    except OracleError as e:
                        rerr = (e.kind, e.msg)
                    pl = bx.Placement("x", dev, np.zeros(m["V"], np.int64), eo, off)
                    try:
                        rep = bx.simulate(gg, pl, caps, bx.CommModel(*cmv), mem, record_trace=True)
                        oerr = None
                    except bx.Error as e:
                        oerr = (e.kind, e.msg)
                    assert oerr == rerr, (gi, n, algo, mem)
                    if rerr is None:
                        assert len(rep.trace) == rcount
                        assert bx.trace_to_csv(rep.trace) == rtext, (gi, n, algo, mem)
                        plain = bx.simulate(gg, pl, caps, bx.CommModel(*cmv), mem)
                        assert plain.makespan_us == rep.makespan_us
                        assert np.array_equal(plain.start_us, rep.start_us)


def test_one_shot_calls_reuse_the_arena(bx):
    """bx_place in steady state: repeated calls of different sizes stay
    exact (the thread's arena is reused and grown, never stale)."""
    for rep in range(3):
        for g in (W.branchy(6, rep), W.layered_dag(20, 40, rep), W.branchy(3, rep + 10)):
            m = W.as_meta_dict(g)
            gg = bx.MetaGraph.from_dict(m)
            caps = [W.bench_capacity(g, 4, 1.3)] * 4
            for cmv in ((12.5, 0.002, 1), (5.0, 0.001, 0)):
                p = bx.place_metf(gg, caps, bx.CommModel(*cmv))
                o = Restate.place(m, 1, caps, cmv)
                assert np.array_equal(p.device_of, o.device_of) and np.array_equal(p.start_us, o.start_us)
                r = bx.simulate(gg, p, caps, bx.CommModel(*cmv))
                s = Restate.simulate(m, caps, cmv, 1, o.device_of, o.exec_order, o.exec_off)
                assert r.makespan_us == s.makespan


def test_plan_simulate_skips_jobs_without_placement(bx):
    """Jobs rejected by host validation or failing in the placer leave empty
    exec lists: simulate reports a validation error for them and the other
    jobs' reports stay exact (no stale lists, no fault)."""
    g = W.branchy(5, 1)
    m = W.as_meta_dict(g)
    gg = bx.MetaGraph.from_dict(m)
    cm = bx.CommModel(12.5, 0.002, 1)
    ok_caps = np.array([W.bench_capacity(g, 3, 1.5)] * 3, np.int64)
    jobs = [bx.Job(0, "m-etf", ok_caps, cm),
            bx.Job(0, "m-etf", np.array([100, -1], np.int64), cm),       # roster error (host)
            bx.Job(0, "m-etf", np.array([10, 10], np.int64), cm),        # fits on no device (placer)
            bx.Job(0, "m-topo", np.array([10, 10], np.int64), cm),       # m-topo cap error
            bx.Job(0, "m-etf", ok_caps, cm)]
    plan = bx.Plan([gg], jobs)
    for _ in range(2):  # twice: the second run starts from the first run's workspace
        plan.upload()
        plan.place()
        plan.download()
        assert [plan.status(i)[0] for i in range(5)] == [0, 2, 3, 3, 0]
        plan.simulate(bx.TRAINING_PERSISTENT)
        reps = plan.sim_download()
        o = Restate.place(m, 1, list(ok_caps), (12.5, 0.002, 1))
        s = Restate.simulate(m, list(ok_caps), (12.5, 0.002, 1), 1, o.device_of, o.exec_order, o.exec_off)
        for i in (0, 4):
            assert reps[i].makespan_us == s.makespan
        for i in (1, 2, 3):
            assert reps[i] == (2, "placement must assign every node exactly once")
    plan.close()


def _tiny_dag(rng, V, p=0.35):
    src, dst = [], []
    for a in range(V):
        for b in range(a + 1, V):
            if rng.random() < p:
                src.append(a)
                dst.append(b)
    o = np.lexsort((dst, src))
    src, dst = np.array(src, np.int32)[o], np.array(dst, np.int32)[o]
    tensor = rng.integers(1, 4000, V)
    return dict(V=V, E=len(src), k=rng.integers(10, 121, V), temp=rng.integers(0, 50, V),
                perm=rng.integers(1, 100, V), out=rng.integers(1, 100, V), esrc=src, edst=dst,
                ebytes=tensor[src].astype(np.int64) if len(src) else np.zeros(0, np.int64))


@needs_ref
def test_oracle_makespan_vs_reference(bx):
    """The exhaustive oracle (oracle.cpp:185-212) on the GPU simulator vs the
    reference's own oracle_makespan: tiny DAGs, 1-3 devices, both comm
    modes, both memory modes, no / loose / tight capacities (memory-skipped
    assignments, and nothing fitting), error texts included."""
    rng = np.random.default_rng(21)
    cases = 0
    for t in range(14):
        V = int(rng.integers(1, 9))
        g = _tiny_dag(rng, V)
        gg = bx.MetaGraph.from_dict(g)
        rg = Ref.graph(W.as_ref_base(g), pipeline=-1)
        need = g["perm"] + g["out"] + g["temp"]
        for n in (1, 2, 3):
            for cm in ((3.0, 0.01, 1), (2.0, 0.02, 0)):
                for cap in (None, int(need.sum()), int(need.max() + need.min())):
                    mm = int(rng.integers(0, 2))
                    try:
                        o = Ref.oracle_makespan(rg, n, cm, cap, mm)
                        oe = None
                    except OracleError as e:
                        o, oe = None, (e.kind, str(e))
                    try:
                        p = bx.oracle_makespan(gg, n, bx.CommModel(*cm), cap, mm)
                        pe = None
                    except bx.Error as e:
                        p, pe = None, (e.kind, e.msg)
                    assert (p, pe) == (o, oe), (t, n, cm, cap, mm)
                    cases += 1
    assert cases == 14 * 3 * 2 * 3
    g = _tiny_dag(rng, 13)
    with pytest.raises(bx.InfeasibleError, match="instance too large: 13 nodes > 12"):
        bx.oracle_makespan(bx.MetaGraph.from_dict(g), 2, bx.CommModel(1.0, 0.0, 1))
    g = _tiny_dag(rng, 6)
    with pytest.raises(bx.InfeasibleError, match="instance too large: 4 devices > 3"):
        bx.oracle_makespan(bx.MetaGraph.from_dict(g), 4, bx.CommModel(1.0, 0.0, 1))
    g = _tiny_dag(rng, 8, p=0.05)
    with pytest.raises(bx.InfeasibleError, match="more than 10 execution orders"):
        bx.oracle_makespan(bx.MetaGraph.from_dict(g), 2, bx.CommModel(1.0, 0.0, 1), max_extensions=10)
