"""GPU: the favourite-child LP (build_lp + solve_relaxed, lp.cpp:14-278).
Eigen3 is absent, so the reference's IPM cannot run here: parity is pinned
at the tolerance of the reference's own LP tests (proj/tests/test_lp.cpp)
plus the LP objective from an independent solver (scipy HiGHS)."""
import numpy as np
import pytest

import kats
from paper_2301_08695_b200 import workloads as W

pytestmark = pytest.mark.gpu
BYTES_ARE_MICROS = (0.0, 1.0, 0)  # test_lp.cpp:13


def meta(bx, g):
    return bx.MetaGraph.from_dict(g)


def lp_rows(g, cm):
    """The reference's rows of G z <= h (lp.cpp:33-77) in numpy."""
    V, E = g["V"], g["E"]
    k = g["k"].astype(float)
    import paper_2301_08695_b200 as bx
    c = np.array([bx.comm_time(bx.CommModel(*cm), b) for b in g["ebytes"]], float)
    nv = V + E + 1
    rows, rhs = [], []

    def row(ents, r):
        v = np.zeros(nv)
        for i, a in ents:
            v[i] += a
        rows.append(v)
        rhs.append(r)
    for i in range(V):
        row([(i, 1), (V + E, -1)], -k[i])
    for e in range(E):
        row([(g["esrc"][e], 1), (g["edst"][e], -1), (V + e, c[e])], -k[g["esrc"][e]])
    for i in range(V):
        es = [e for e in range(E) if g["esrc"][e] == i]
        if es:
            row([(V + e, -1) for e in es], 1 - len(es))
    for j in range(V):
        es = [e for e in range(E) if g["edst"][e] == j]
        if es:
            row([(V + e, -1) for e in es], 1 - len(es))
    return np.array(rows), np.array(rhs), c


def test_row_counts_diamond(bx):  # test_lp.cpp:53-60
    sol = bx.solve_relaxed(meta(bx, kats.diamond(2, 8)), bx.CommModel(*BYTES_ARE_MICROS))
    r = sol.rows
    assert (r["completion"], r["precedence"], r["child"], r["parent"]) == (4, 4, 3, 3)
    assert r["bound"] == 4 + 1 + 2 * 4


def test_single_node(bx):  # :62-70
    sol = bx.solve_relaxed(meta(bx, kats.graph([kats.node(0, 9)], [])), bx.CommModel(*BYTES_ARE_MICROS))
    assert sol.w == pytest.approx(9.0, rel=1e-4)


def test_two_node_chain(bx):  # :72-93
    g = kats.graph([kats.node(0, 10), kats.node(1, 10)], [(0, 1, 8)])
    sol = bx.solve_relaxed(meta(bx, g), bx.CommModel(*BYTES_ARE_MICROS))
    assert sol.x[0] < 0.1
    assert sol.w == pytest.approx(20.0, rel=1e-3)
    best = min(10.0 + 8.0 * (i / 1000) + 10.0 for i in range(1001))
    assert sol.w <= best + 1e-2


def test_at_most_one_child(bx):  # :95-103
    g = kats.graph([kats.node(i, 10) for i in range(3)], [(0, 1, 8), (0, 2, 8)])
    sol = bx.solve_relaxed(meta(bx, g), bx.CommModel(*BYTES_ARE_MICROS))
    assert sol.x[0] + sol.x[1] >= 1.0 - 1e-6


def test_no_edges(bx):  # :105-111
    g = kats.graph([kats.node(0, 4), kats.node(1, 11), kats.node(2, 7)], [])
    assert bx.solve_relaxed(meta(bx, g), bx.CommModel(*BYTES_ARE_MICROS)).w == pytest.approx(11.0, rel=1e-4)


@pytest.mark.parametrize("seed", range(12))
def test_feasible_bounded_deterministic_and_optimal(bx, seed):
    """:113-130 (primal feasible at 1e-6, w <= the all-ones objective,
    deterministic) plus the optimum of an independent solver (HiGHS)."""
    from scipy.optimize import linprog
    rng = np.random.default_rng(seed)
    V = int(rng.integers(3, 15))
    nodes = [kats.node(i, int(rng.integers(1, 121))) for i in range(V)]
    edges = sorted({(int(a), int(b)) for a, b in rng.integers(0, V, (2 * V, 2)) if a < b})
    g = kats.graph(nodes, [(a, b, int(rng.integers(0, 61))) for a, b in edges])
    cm = bx.CommModel(*BYTES_ARE_MICROS)
    sol = bx.solve_relaxed(meta(bx, g), cm)
    again = bx.solve_relaxed(meta(bx, g), cm)
    assert sol.w == again.w and np.array_equal(sol.x, again.x)
    A, b, c = lp_rows(g, BYTES_ARE_MICROS)
    z = np.concatenate([sol.s, sol.x, [sol.w]])
    assert np.all(A @ z <= b + 1e-6)
    assert np.all(sol.s >= -1e-9) and np.all((sol.x >= 0) & (sol.x <= 1))
    # all-ones objective: longest path with every transfer paid
    start = np.zeros(V)
    for e in np.argsort(g["edst"], kind="stable"):
        s_, d_ = g["esrc"][e], g["edst"][e]
    order = list(range(V))  # ids ascending are topological here (edges a < b)
    w1 = 0.0
    for u in order:
        for e in range(g["E"]):
            if g["edst"][e] == u:
                start[u] = max(start[u], start[g["esrc"][e]] + g["k"][g["esrc"][e]] + c[e])
        w1 = max(w1, start[u] + g["k"][u])
    assert sol.w <= w1 + 1e-6
    obj = np.zeros(V + g["E"] + 1)
    obj[-1] = 1
    bounds = [(0, None)] * V + [(0, 1)] * g["E"] + [(0, None)]
    ref = linprog(obj, A_ub=A, b_ub=b, bounds=bounds, method="highs")
    assert ref.status == 0
    assert sol.w == pytest.approx(ref.fun, rel=1e-4, abs=1e-3)


def test_fig2_makespans_through_lp(bx):
    """test_placers.cpp:190-225: the paper's Fig. 2 instance through the LP
    (run_placer's m-SCT path): makespan 8 unlimited, 9 at capacity 4."""
    g = kats.graph([kats.node(0, 4, 0, 2, 0), kats.node(1, 1, 0, 1, 0), kats.node(2, 4, 0, 2, 0),
                    kats.node(3, 1, 0, 1, 0), kats.node(4, 4, 0, 1, 0), kats.node(5, 1, 0, 1, 0)],
                   [(0, 3, 2), (0, 4, 3), (1, 2, 3), (1, 5, 2)])
    gg = meta(bx, g)
    cm = bx.CommModel(0.0, 1.0, 1)

    def run(cap):
        p = bx.run_msct(gg, [cap, cap], cm)
        return bx.simulate(gg, p, [cap, cap], cm, bx.TRAINING_PERSISTENT)
    unl = run(1 << 20)
    assert unl.makespan_us == 8 and max(unl.peak_bytes) > 4
    capped = run(4)
    assert capped.makespan_us == 9 and max(capped.peak_bytes) <= 4


def test_c3_transformer_lp_end_to_end(bx):
    """Config C3 with the LP (no fixed fav map): ingest -> LP -> favourites
    -> m-SCT on the GPU; objective cross-checked against HiGHS on the same
    rows, placement verified by the simulator."""
    from scipy.optimize import linprog
    from scipy.sparse import lil_matrix
    gen, n, _, kw, f = W.CONFIGS["C3_transformer_msct_tight"]
    mg, _ = bx.build_grouped(gen(), **kw)
    cm = bx.CommModel(*W.COMM_TEST)
    fc, fp, st, sol = bx.sct_favorites(mg, cm)
    assert sol.iterations < 200 and st[0] > 0
    cap = W.meta_capacity(mg, n, f)
    p = bx.place_msct(mg, [cap] * n, cm, fc)
    ok, diag, rep = bx.verify_placement(mg, p, [cap] * n, cm, bx.TRAINING_PERSISTENT)
    assert ok, diag
    V, E = mg.V, mg.E
    c = np.array([bx.comm_time(cm, b) for b in mg.ebytes], float)
    A = lil_matrix((V + E + 2 * V, V + E + 1))
    b = []
    r = 0
    for i in range(V):
        A[r, i], A[r, V + E] = 1, -1
        b.append(-mg.k[i])
        r += 1
    for e in range(E):
        A[r, mg.esrc[e]], A[r, mg.edst[e]], A[r, V + e] = 1, -1, c[e]
        b.append(-mg.k[mg.esrc[e]])
        r += 1
    for i in range(V):
        lo, hi = mg.out_off[i], mg.out_off[i + 1]
        if hi > lo:
            for e in range(lo, hi):
                A[r, V + e] = -1
            b.append(1 - (hi - lo))
            r += 1
    for j in range(V):
        lo, hi = mg.in_off[j], mg.in_off[j + 1]
        if hi > lo:
            for x in range(lo, hi):
                A[r, V + mg.in_edge[x]] = -1
            b.append(1 - (hi - lo))
            r += 1
    A = A[:r].tocsr()
    obj = np.zeros(V + E + 1)
    obj[-1] = 1
    ref = linprog(obj, A_ub=A, b_ub=np.array(b, float),
                  bounds=[(0, None)] * V + [(0, 1)] * E + [(0, None)], method="highs")
    assert ref.status == 0
    assert sol.w == pytest.approx(ref.fun, rel=1e-4)


def _highs_objective(mg, cm):
    """build_lp's rows (lp.cpp:14-79, unscaled) solved by HiGHS."""
    from scipy.optimize import linprog
    import scipy.sparse as sp
    V, E = mg.V, mg.E
    c = np.array([bx_comm(cm, b) for b in mg.ebytes], float)
    rows, cols, vals, b = [], [], [], []
    r = 0
    for i in range(V):
        rows += [r, r]
        cols += [i, V + E]
        vals += [1, -1]
        b.append(-mg.k[i])
        r += 1
    for e in range(E):
        rows += [r, r, r]
        cols += [mg.esrc[e], mg.edst[e], V + e]
        vals += [1, -1, c[e]]
        b.append(-mg.k[mg.esrc[e]])
        r += 1
    for off, ids in ((mg.out_off, None), (mg.in_off, mg.in_edge)):
        for i in range(V):
            lo, hi = off[i], off[i + 1]
            if hi > lo:
                for x in range(lo, hi):
                    rows.append(r)
                    cols.append(V + (x if ids is None else ids[x]))
                    vals.append(-1)
                b.append(1 - (hi - lo))
                r += 1
    A = sp.csr_matrix((vals, (rows, cols)), shape=(r, V + E + 1))
    obj = np.zeros(V + E + 1)
    obj[-1] = 1
    ref = linprog(obj, A_ub=A, b_ub=np.array(b, float), bounds=[(0, None)] * V + [(0, 1)] * E + [(0, None)],
                  method="highs")
    assert ref.status == 0
    return ref.fun


def bx_comm(cm, b):
    import paper_2301_08695_b200 as bx
    return bx.comm_time(cm, b)


@pytest.mark.parametrize("name", ["C1_inception_mtopo_metf", "C2_gnmt_metf_coplace"])
def test_model_config_lps_match_highs(bx, name):
    """The device IPM (K5) on the C1 and C2 meta graphs (10.8k / 26.5k LP
    variables): level-scheduled left-looking factor with warp-summed long
    update lists, and on C2 the dense tail block (the ordering's final 507
    columns); objective = HiGHS on the same rows."""
    gen, n, _, kw, f = W.CONFIGS[name]
    mg, _ = bx.build_grouped(gen(), **kw)
    cm = bx.CommModel(*W.COMM_TEST)
    sol = bx.solve_relaxed(mg, cm)
    assert sol.iterations < 200 and sol.solver["update_pairs"] > 0
    assert sol.w == pytest.approx(_highs_objective(mg, cm), rel=1e-4)
