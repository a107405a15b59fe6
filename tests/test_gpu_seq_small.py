"""GPU parity of K2q (csrc/seqsmall.cu), the small-frontier placer for
sequential comm mode, against the C restatement: seeded graphs x rosters x
comm models, mixed byte counts (cache hits change the tail fold), nodes with
more than the 8 recorded parents, memory discards, device exclusions and
infeasible errors, plus the hand-offs to the general kernels (a frontier
wider than 512 pairs at the start or mid-run). Bit-exact."""
import numpy as np
import pytest

from oracle import OracleError, Restate
from paper_2301_08695_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _plan_one(bx, gg, algo, caps, cm, options=None):
    plan = bx.Plan([gg], [bx.Job(0, algo, np.asarray(caps, np.int64), cm, None)], options=options)
    plan.upload()
    plan.place()
    plan.download()
    st, msg = plan.status(0)
    kern = plan.job_kernel(0)
    p = plan.result(0) if st == 0 else None
    plan.close()
    return st, msg, p, kern


def _oracle(m, caps, cm):
    try:
        return Restate.place(m, 1, caps, cm, None), None
    except OracleError as e:
        return None, (e.kind, e.msg)


def _same(p, o):
    assert np.array_equal(p.device_of, o.device_of)
    assert np.array_equal(p.start_us, o.start_us)
    assert np.array_equal(p.exec_order_flat, o.exec_order)
    assert np.array_equal(p.exec_off, o.exec_off)
    assert list(p.stats) == list(o.stats)


def _mixed_bytes(m, seed):
    rng = np.random.default_rng(seed)
    m = dict(m)
    m["ebytes"] = rng.integers(1, 200_000, len(m["esrc"])).astype(np.int64)
    return m


def _fan_in(seed, width=12, depth=6):
    """Layers of `width` nodes, every node of a layer feeding a join node with
    `width` parents (more than K2q records per slot), the join feeding the
    next layer."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    V = 0
    prev = None
    for _ in range(depth):
        layer = list(range(V, V + width))
        V += width
        if prev is not None:
            for x in layer:
                src.append(prev)
                dst.append(x)
        join = V
        V += 1
        for x in layer:
            src.append(x)
            dst.append(join)
        prev = join
    order = np.lexsort((dst, src))
    return dict(V=V, E=len(src), k=rng.integers(10, 300, V).astype(np.int64),
                temp=rng.integers(0, 1000, V).astype(np.int64), perm=rng.integers(1000, 5000, V).astype(np.int64),
                out=rng.integers(1000, 5000, V).astype(np.int64), esrc=np.array(src, np.int32)[order],
                edst=np.array(dst, np.int32)[order], ebytes=rng.integers(1000, 90000, len(src)).astype(np.int64)[order])


def _graphs():
    out = []
    for seed in range(3):
        out.append(("branchy", W.as_meta_dict(W.branchy(8, seed))))
        out.append(("grid", W.as_meta_dict(W.grid_chain(30, 4, seed))))
        out.append(("grid_mixed", _mixed_bytes(W.as_meta_dict(W.grid_chain(25, 5, seed)), seed)))
        out.append(("fan_in", _fan_in(seed)))
    return out


@pytest.mark.parametrize("idx", range(12))
def test_seq_small_vs_oracle(bx, idx):
    name, m = _graphs()[idx]
    gg = bx.MetaGraph.from_dict(m)
    rng = np.random.default_rng(100 + idx)
    need = m["perm"] + m["out"] + m["temp"]
    used = 0
    for n in (1, 2, 3, 4, 7, 8, 16, 32):
        for f in (0.9, 1.0, 1.05, 1.6):
            cap = int(np.ceil((need.sum() / n + need.max()) * f))
            caps = [int(cap * rng.uniform(0.75, 1.1)) for _ in range(n)]
            for cmv in ((5.0, 0.001, 0), (0.0, 0.0, 0), (40.0, 0.01, 0)):
                o, oe = _oracle(m, caps, cmv)
                st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(*cmv))
                assert (None if st == 0 else (st, msg)) == oe, (name, n, f, cmv, kern)
                if oe is None:
                    _same(p, o)
                used += kern == "seq-small"
    assert used > 0, "K2q never ran"


def test_seq_small_matches_the_cta_kernel(bx):
    """The same sequential placements through K2q and through the 8-warp
    kernel it replaces for small frontiers."""
    for seed in range(3):
        m = W.as_meta_dict(W.grid_chain(200, 3, seed))
        gg = bx.MetaGraph.from_dict(m)
        need = m["perm"] + m["out"] + m["temp"]
        for n in (2, 4, 8):
            caps = [int((need.sum() / n + need.max()) * 1.1)] * n
            a = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(5.0, 0.001, 0))
            b = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(5.0, 0.001, 0),
                          options={"wide_min_vn": 0, "no_small_frontier": 1})
            assert a[0] == 0 and b[0] == 0 and a[3] == "seq-small" and b[3] == "cta-seq"
            pa, pb = a[2], b[2]
            assert np.array_equal(pa.device_of, pb.device_of) and np.array_equal(pa.start_us, pb.start_us)
            assert np.array_equal(pa.exec_order_flat, pb.exec_order_flat)
            assert np.array_equal(pa.exec_off, pb.exec_off) and list(pa.stats) == list(pb.stats)


def test_seq_small_wide_start_hands_off(bx):
    """300 sources x 4 devices (1200 pairs > 512) joined by one sink with 300
    parents: the general kernel places it."""
    rng = np.random.default_rng(3)
    srcs = 300
    V = srcs + 1
    src = list(range(srcs))
    dst = [srcs] * srcs
    m = dict(V=V, E=srcs, k=rng.integers(50, 150, V).astype(np.int64),
             temp=rng.integers(0, 1000, V).astype(np.int64), perm=rng.integers(1000, 5000, V).astype(np.int64),
             out=rng.integers(1000, 5000, V).astype(np.int64), esrc=np.array(src, np.int32),
             edst=np.array(dst, np.int32), ebytes=rng.integers(1000, 60000, srcs).astype(np.int64))
    gg = bx.MetaGraph.from_dict(m)
    need = m["perm"] + m["out"] + m["temp"]
    caps = [int((need.sum() / 4 + need.max()) * 1.3)] * 4
    o, oe = _oracle(m, caps, (5.0, 0.001, 0))
    st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(5.0, 0.001, 0))
    assert oe is None and st == 0
    _same(p, o)
    assert kern != "seq-small"


def test_seq_small_midrun_overflow_hands_off(bx):
    """A chain fanning out to 400 children mid-run: K2q starts, overflows,
    and the general kernel restarts the job from scratch (K2q's cache rows
    live in its own array, so the general kernel's cache is untouched)."""
    rng = np.random.default_rng(5)
    chain, fan = 20, 400
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
        o, oe = _oracle(m, caps, (5.0, 0.001, 0))
        st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(5.0, 0.001, 0))
        assert oe is None and st == 0
        _same(p, o)
        assert kern != "seq-small", kern


def test_seq_small_wide_times(bx):
    """Compute times whose sum passes 2^31 us: K2q keeps int64 times (no
    range hand-off, unlike K2s), results stay exact."""
    for seed in range(2):
        m = W.as_meta_dict(W.branchy(6, seed))
        m["k"] = m["k"] * 20_000_000
        gg = bx.MetaGraph.from_dict(m)
        need = m["perm"] + m["out"] + m["temp"]
        for n in (2, 4):
            caps = [int((need.sum() / n + need.max()) * 1.1)] * n
            o, oe = _oracle(m, caps, (5.0, 0.001, 0))
            st, msg, p, kern = _plan_one(bx, gg, "m-etf", caps, bx.CommModel(5.0, 0.001, 0))
            assert oe is None and st == 0
            _same(p, o)
            assert kern == "seq-small", kern
