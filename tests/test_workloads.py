"""CPU: the synthetic workload generators emit valid reference graphs
(make_graph accepts them, singleton grouping is the identity) and the
capacity rule matches the reference's bench_capacity."""
import numpy as np
import pytest

from oracle import Ref
from paper_2301_08695_b200 import workloads as W

GENS = [lambda s: W.layered_dag(10, 12, s), lambda s: W.layered_dag_fast(20, 30, s),
        lambda s: W.grid_chain(25, 8, s), lambda s: W.branchy(8, s), lambda s: W.wide_random(300, s)]


@pytest.mark.parametrize("gi", range(len(GENS)))
def test_generator_invariants(gi):
    for seed in range(3):
        g = GENS[gi](seed)
        V = g["V"]
        s, d = g["esrc"].astype(np.int64), g["edst"].astype(np.int64)
        assert np.all(s < d) and np.all(d < V)
        key = s * V + d
        assert np.all(np.diff(key) > 0), "sorted by (src, dst), unique"
        assert np.all(g["k"] >= 50) and np.all(g["k"] <= 150)
        assert np.all(g["ebytes"] >= 1024) and np.all(g["ebytes"] <= 65536)
        again = GENS[gi](seed)
        assert all(np.array_equal(g[k], again[k]) for k in ("k", "esrc", "edst", "ebytes", "perm"))


@pytest.mark.skipif(not Ref.available(), reason="reference not compiled on this host")
@pytest.mark.parametrize("gi", range(len(GENS)))
def test_generator_graphs_are_reference_graphs(gi):
    g = GENS[gi](1)
    rg = Ref.graph(W.as_ref_base(g), -1)
    m = rg.meta()
    assert np.array_equal(m["esrc"], g["esrc"]) and np.array_equal(m["edst"], g["edst"])
    assert np.array_equal(m["k"], g["k"]) and np.array_equal(m["ebytes"], g["ebytes"])
    for n in (2, 4, 16):
        for f in (1.05, 1.5):
            assert W.bench_capacity(g, n, f) == Ref.bench_capacity(rg, n, f)


def test_sweep_shape():
    gs = W.sweep_graphs(0, 8, vmin=200, vmax=400)
    jobs = W.sweep_jobs(gs)
    assert len(gs) == 8 and len(jobs) == 8 * 4 * 16
    assert {n for _, n, _ in jobs} == {2, 4, 8, 16}
    other = W.sweep_graphs(1, 8, vmin=200, vmax=400)
    assert not np.array_equal(gs[0]["esrc"], other[0]["esrc"]) or gs[0]["V"] != other[0]["V"]
