"""CPU: the host ingest (make_graph + colocation / co-placement / fusion,
csrc/ingest.cpp) against the reference's own transforms (oracle/_ref) on
seeded graphs, the committed ingest golden vectors, and the reference's
validation error texts (proj/src/graph.cpp:99-194, transforms.cpp:329-351)."""
import json
import os

import numpy as np
import pytest

import paper_2301_08695_b200 as bx
from oracle import OracleError, Ref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PIPES = {-1: dict(singleton=True), 0: dict(coplacement=False, fusion=False),
         2: dict(coplacement=True, fusion=False), 4: dict(coplacement=False, fusion=True),
         6: dict(coplacement=True, fusion=True)}


def _cmp(meta, grouping, r):
    assert meta.V == r["V"] and meta.E == r["E"]
    for a, b in ((meta.k, "k"), (meta.temp, "temp"), (meta.perm, "perm"), (meta.out, "out"),
                 (meta.esrc, "esrc"), (meta.edst, "edst"), (meta.ebytes, "ebytes")):
        assert np.array_equal(a, r[b]), b
    assert np.array_equal(grouping["group_of"], r["group_of"])
    assert np.array_equal(grouping["edge_base_count"], r["ecount"])
    assert np.array_equal(grouping["member_off"], r["member_off"])
    assert np.array_equal(grouping["members"], r["members"])
    assert np.array_equal(meta.first_id, r["first_id"])


def node_graph(nodes, edges, coloc=None, pairs=None):
    n = len(nodes)
    has_pair = np.zeros(n, np.uint8)
    pair = np.zeros(n, np.int64)
    for i, p in (pairs or {}).items():
        has_pair[i], pair[i] = 1, p
    return dict(id=np.array([x[0] for x in nodes], np.int64), k=np.array([x[1] for x in nodes], np.int64),
                temp=np.array([x[2] for x in nodes], np.int64), perm=np.array([x[3] for x in nodes], np.int64),
                out=np.array([x[4] for x in nodes], np.int64),
                coloc=np.array(coloc if coloc is not None else [-1] * n, np.int32), has_pair=has_pair, pair=pair,
                src=np.array([e[0] for e in edges], np.int64), dst=np.array([e[1] for e in edges], np.int64),
                bytes=np.array([e[2] for e in edges], np.int64))


# proj/tests/test_graph.cpp / graph.cpp:99-194 validation texts
ERROR_CASES = [
    ("duplicate id", node_graph([(1, 1, 0, 0, 0), (1, 2, 0, 0, 0)], []), "duplicate node id 1"),
    ("negative field", node_graph([(0, -1, 0, 0, 0)], []), "node 0 has a negative field"),
    ("self pair", node_graph([(0, 1, 0, 0, 0)], [], pairs={0: 0}), "node 0 coplace_pair references itself"),
    ("asymmetric pair", node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0)], [], pairs={0: 1}),
     "coplace_pair between 0 and 1 is not symmetric"),
    ("dangling pair", node_graph([(0, 1, 0, 0, 0)], [], pairs={0: 9}), "dangling reference: unknown node id 9"),
    ("negative bytes", node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0)], [(0, 1, -5)]), "edge 0->1 has negative bytes"),
    ("self edge", node_graph([(0, 1, 0, 0, 0)], [(0, 0, 1)]), "self edge on node 0"),
    ("dangling edge", node_graph([(0, 1, 0, 0, 0)], [(0, 7, 1)]), "dangling reference: unknown node id 7"),
    ("duplicate edge", node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0)], [(0, 1, 1), (0, 1, 2)]),
     "duplicate edge 0->1"),
    ("cycle", node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0), (2, 1, 0, 0, 0)], [(0, 1, 1), (1, 2, 1), (2, 1, 1)]),
     "graph has a cycle through node ids {1, 2}"),
    ("colocation cycle", node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0), (2, 1, 0, 0, 0)], [(0, 1, 1), (1, 2, 1)],
                                    coloc=[5, -1, 5]),
     "colocation-induced cycle: meta graph is cyclic; groups of base node ids {0, 1} remain"),
]


@pytest.mark.parametrize("name,g,msg", ERROR_CASES, ids=[c[0] for c in ERROR_CASES])
def test_ingest_validation_texts(name, g, msg):
    with pytest.raises(bx.ValidationError) as ei:
        bx.build_grouped(g)
    assert ei.value.msg == msg
    if Ref.available():
        with pytest.raises(OracleError) as er:
            Ref.graph(g, 6)
        assert er.value.kind == 2 and er.value.msg == msg


def test_coplacement_skips_cycle_closing_pair():
    # 0 -> 1 -> 2 plus pair (0, 2): contracting would close 0~>2 besides any
    # direct edge, so the pair is skipped (transforms.cpp:359-370) and the
    # chain then merges through the out-degree-1 rule
    g = node_graph([(0, 1, 0, 0, 0), (1, 1, 0, 0, 0), (2, 1, 0, 0, 0), (3, 1, 0, 0, 0)],
                   [(0, 1, 1), (1, 2, 1), (0, 3, 1)], pairs={0: 2, 2: 0})
    m, gr = bx.build_grouped(g, coplacement=True, fusion=False)
    if Ref.available():
        _cmp(m, gr, Ref.graph(g, 2).meta())


@pytest.mark.skipif(not Ref.available(), reason="reference not compiled on this host")
@pytest.mark.parametrize("seed", range(12))
def test_ingest_matches_reference_transforms(seed):
    fam = ["branchy", "layered-chain", "random-dag"][seed % 3]
    g = Ref.generate(fam, 150 + 20 * seed, 500 + seed, layers=5, edge_prob=0.05,
                     colocate_edge_frac=[0.0, 0.1, 0.3][seed % 3], coplace_frac=[0.05, 0.2, 0.0][seed % 3])
    for pipe, kw in PIPES.items():
        try:
            r = Ref.graph(g, pipe).meta()
        except OracleError as e:
            with pytest.raises(bx.ValidationError) as ei:
                bx.build_grouped(g, **kw)
            assert ei.value.msg == e.msg
            continue
        m, gr = bx.build_grouped(g, **kw)
        _cmp(m, gr, r)


def test_ingest_golden_vectors():
    z = np.load(os.path.join(GOLD, "ingest.npz"))
    index = json.load(open(os.path.join(GOLD, "ingest_index.json")))
    for rec in index:
        c = rec["case"]
        g = {k: z[f"c{c}_in_{k}"] for k in ("id", "k", "temp", "perm", "out", "coloc", "has_pair", "pair", "src",
                                            "dst", "bytes")}
        m, gr = bx.build_grouped(g, **PIPES[rec["pipe"]])
        r = {k: z[f"c{c}_out_{k}"] for k in ("k", "temp", "perm", "out", "esrc", "edst", "ebytes", "group_of",
                                             "ecount", "member_off", "members", "first_id")}
        r["V"], r["E"] = len(r["k"]), len(r["esrc"])
        _cmp(m, gr, r)


@pytest.mark.skipif(not Ref.available(), reason="reference not compiled on this host")
@pytest.mark.parametrize("fam,V,frac,coloc", [("layered-chain", 12000, 0.05, 0.0), ("branchy", 6000, 0.2, 0.05),
                                               ("layered-chain", 8000, 0.3, 0.02)])
def test_ingest_at_scale_matches_reference(fam, V, frac, coloc):
    """Level-pruned co-placement path checks and fusion at thousands of
    nodes: identical meta graphs and groupings to the reference transforms."""
    g = Ref.generate(fam, V, 77, layers=60, coplace_frac=frac, colocate_edge_frac=coloc)
    for pipe in (2, 6):
        try:
            r = Ref.graph(g, pipe).meta()
        except OracleError as e:
            with pytest.raises(bx.ValidationError) as ei:
                bx.build_grouped(g, **PIPES[pipe])
            assert ei.value.msg == e.msg
            continue
        m, gr = bx.build_grouped(g, **PIPES[pipe])
        _cmp(m, gr, r)
