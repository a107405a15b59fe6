"""GPU parity of the small-frontier placer K2s (csrc/smallsched.cu) against
the C restatement: seeded graphs x rosters x algorithms, non-uniform edge
byte counts (the shared-memory cache rows), memory discards, device
exclusions and infeasible errors, plus every hand-off to the general
kernels (frontier wider than 256 pairs at the start or mid-run, values
outside the int32 bound). Bit-exact."""
import numpy as np
import pytest

import golden_cases
from oracle import OracleError, Restate
from paper_2301_08695_b200 import workloads as W

pytestmark = pytest.mark.gpu
ALGO = ["m-topo", "m-etf", "m-sct"]


def _plan_one(bx, gg, algo, caps, cm, fav=None, options=None):
    plan = bx.Plan([gg], [bx.Job(0, algo, np.asarray(caps, np.int64), cm, fav)], options=options)
    plan.upload()
    plan.place()
    plan.download()
    st, msg = plan.status(0)
    kern = plan.job_kernel(0)
    p = plan.result(0) if st == 0 else None
    plan.close()
    return st, msg, p, kern


def _oracle(m, algo, caps, cm, fav):
    try:
        return Restate.place(m, algo, caps, cm, fav), None
    except OracleError as e:
        return None, (e.kind, e.msg)


def _same(p, o):
    assert np.array_equal(p.device_of, o.device_of)
    assert np.array_equal(p.start_us, o.start_us)
    assert np.array_equal(p.exec_order_flat, o.exec_order)
    assert np.array_equal(p.exec_off, o.exec_off)
    assert list(p.stats) == list(o.stats)


def _mixed_bytes(g, seed):
    """Per-edge byte counts (different on a producer's out-edges), so many
    producers need K2s's cache rows."""
    rng = np.random.default_rng(seed)
    m = W.as_meta_dict(g)
    m["ebytes"] = rng.integers(1, 200_000, len(m["esrc"])).astype(np.int64)
    return m


def _graphs():
    out = []
    for seed in range(4):
        out.append(("branchy", W.as_meta_dict(W.branchy(8, seed))))
        out.append(("grid", W.as_meta_dict(W.grid_chain(30, 4, seed))))
        out.append(("grid_mixed", _mixed_bytes(W.grid_chain(25, 5, seed), seed)))
        out.append(("branchy_mixed", _mixed_bytes(W.branchy(6, seed + 10), seed)))
    return out


@pytest.mark.parametrize("idx", range(16))
def test_small_frontier_vs_oracle(bx, idx):
    name, m = _graphs()[idx]
    gg = bx.MetaGraph.from_dict(m)
    fav = golden_cases.fav_first(m)
    rng = np.random.default_rng(idx)
    need = m["perm"] + m["out"] + m["temp"]
    used = 0
    for n in (1, 2, 3, 4, 7, 8, 16, 32):
        for f in (0.9, 1.0, 1.05, 1.6):
            cap = int(np.ceil((need.sum() / n + need.max()) * f))
            caps = [int(cap * rng.uniform(0.75, 1.1)) for _ in range(n)]
            for cmv in ((12.5, 0.002, 1), (0.0, 0.0, 1), (40.0, 0.01, 1)):
                for algo in (1, 2):
                    fv = fav if algo == 2 else None
                    o, oe = _oracle(m, algo, caps, cmv, fv)
                    st, msg, p, kern = _plan_one(bx, gg, ALGO[algo], caps, bx.CommModel(*cmv), fv)
                    assert (None if st == 0 else (st, msg)) == oe, (name, n, f, cmv, algo, kern)
                    if oe is None:
                        _same(p, o)
                    used += kern == "small-frontier"
    assert used > 0, "the small-frontier kernel never ran"


def test_small_frontier_takes_the_model_configs(bx):
    """C1-C3 meta graphs are placed by K2s (the dispatch the bench measures)."""
    for name in W.CONFIGS:
        gen, n, algos, kw, f = W.CONFIGS[name]
        meta, _ = bx.build_grouped(gen(), **kw)
        cap = W.meta_capacity(meta, n, f)
        m = dict(V=meta.V, E=meta.E, esrc=meta.esrc, edst=meta.edst)
        for algo in algos:
            if algo == "m-topo":
                continue
            fv = golden_cases.fav_first(m) if algo == "m-sct" else None
            st, msg, p, kern = _plan_one(bx, meta, algo, [cap] * n, bx.CommModel(*W.COMM_TEST), fv)
            assert st == 0, msg
            assert kern == "small-frontier", (name, algo, kern)


def test_wide_frontier_hands_off(bx):
    """300 sources x 4 devices (1200 pairs > 256): the general kernel places it."""
    g = W.wide_random(600, 3)
    m = W.as_meta_dict(g)
    V = m["V"]
    gg = bx.MetaGraph.from_dict(m)
    caps = [W.bench_capacity(g, 4, 1.3)] * 4
    o, oe = _oracle(m, 1, caps, W.COMM_TEST, None)
    st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*W.COMM_TEST))
    assert oe is None and st == 0
    _same(p, o)
    srcs = int((np.bincount(m["edst"], minlength=V) == 0).sum())
    if srcs * 4 > 256:
        assert kern != "small-frontier"


def test_midrun_overflow_hands_off(bx):
    """A chain that fans out to 400 children mid-run: K2s starts, overflows,
    and the general kernel restarts the job from scratch."""
    rng = np.random.default_rng(5)
    chain = 20
    fan = 400
    V = chain + fan + 1
    src = list(range(chain - 1)) + [chain - 1] * fan + list(range(chain, chain + fan))
    dst = list(range(1, chain)) + list(range(chain, chain + fan)) + [V - 1] * fan
    order = np.lexsort((dst, src))
    m = dict(V=V, E=len(src), k=rng.integers(50, 150, V).astype(np.int64),
             temp=rng.integers(0, 1000, V).astype(np.int64), perm=rng.integers(1000, 5000, V).astype(np.int64),
             out=rng.integers(1000, 5000, V).astype(np.int64), esrc=np.array(src, np.int32)[order],
             edst=np.array(dst, np.int32)[order], ebytes=rng.integers(1000, 60000, len(src)).astype(np.int64)[order])
    gg = bx.MetaGraph.from_dict(m)
    need = m["perm"] + m["out"] + m["temp"]
    for n in (2, 4):
        caps = [int((need.sum() / n + need.max()) * 1.2)] * n
        o, oe = _oracle(m, 1, caps, W.COMM_TEST, None)
        st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*W.COMM_TEST))
        assert oe is None and st == 0
        _same(p, o)
        assert kern == "rounds", kern


def test_int32_bound_hands_off(bx):
    """Compute times whose sum passes 2^31 us: K2s declines, results stay exact."""
    g = W.branchy(6, 1)
    m = W.as_meta_dict(g)
    m["k"] = m["k"] * 20_000_000
    gg = bx.MetaGraph.from_dict(m)
    caps = [W.bench_capacity(g, 4, 1.2)] * 4
    o, oe = _oracle(m, 1, caps, W.COMM_TEST, None)
    st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*W.COMM_TEST))
    assert oe is None and st == 0
    _same(p, o)
    assert kern != "small-frontier"


def test_small_frontier_can_be_disabled(bx):
    g = W.branchy(10, 2)
    m = W.as_meta_dict(g)
    gg = bx.MetaGraph.from_dict(m)
    caps = [W.bench_capacity(g, 4, 1.1)] * 4
    a = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*W.COMM_TEST))
    b = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*W.COMM_TEST), options={"no_small_frontier": 1})
    assert a[3] == "small-frontier" and b[3] == "rounds"
    assert a[2] == b[2] and a[2].stats == b[2].stats


@pytest.mark.parametrize("which", ["smem", "global"])
def test_small_frontier_up_to_64_devices(bx, which):
    """K2s takes 33-64 devices for m-ETF when no producer needs cache rows
    (pairs pack the device in 6 bits, at most 32 commits per round), with its
    node state in shared memory or (graphs past it) in HBM; graphs with mixed
    byte counts and m-SCT stay at 32 and hand off. Against the restatement,
    tight capacities (discards, exclusions) included."""
    if which == "smem":
        graphs = [W.as_meta_dict(W.grid_chain(40, 3, 1)), W.as_meta_dict(W.branchy(6, 2))]
    else:  # node state past shared memory: 16k+ nodes
        graphs = [W.as_meta_dict(W.grid_chain(5000, 4, 3))]
    rng = np.random.default_rng(9)
    took = 0
    for m in graphs:
        gg = bx.MetaGraph.from_dict(m)
        need = m["perm"] + m["out"] + m["temp"]
        for n in (33, 40, 64):
            for f in (0.95, 1.05, 1.6):
                cap = int(np.ceil((need.sum() / n + need.max()) * f))
                caps = [int(cap * rng.uniform(0.8, 1.1)) for _ in range(n)]
                cmv = (12.5, 0.002, 1)
                o, oe = _oracle(m, 1, caps, cmv, None)
                st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*cmv))
                assert (None if st == 0 else (st, msg)) == oe, (n, f)
                if oe is None:
                    _same(p, o)
                took += kern == "small-frontier"
    assert took > 0
    # mixed bytes at 40 devices: cache rows needed, so the general kernels place it
    m = _mixed_bytes(W.grid_chain(30, 3, 5), 5)
    gg = bx.MetaGraph.from_dict(m)
    need = m["perm"] + m["out"] + m["temp"]
    caps = [int(np.ceil((need.sum() / 40 + need.max()) * 1.3))] * 40
    o, _ = _oracle(m, 1, caps, (12.5, 0.002, 1), None)
    st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(12.5, 0.002, 1))
    assert st == 0 and kern != "small-frontier"
    _same(p, o)
