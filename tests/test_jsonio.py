"""CPU: interchange IO (csrc/jsonio.cpp) against the compiled reference
(oracle/_ref): comm-model JSON (cost_model.cpp:71-134), graph JSON
(graph.cpp:196-309), placement JSON (placers.cpp:367-432) and the binary
CSR sidecar. Emitted texts are compared byte for byte; error kinds and
messages exactly (malformed-JSON syntax errors: kind and prefix only)."""
import json
import os

import numpy as np
import pytest

import paper_2301_08695_b200 as bx
from oracle import OracleError, Ref

pytestmark = pytest.mark.skipif(not Ref.available(), reason="compiled reference (oracle/_ref) missing")

REF_COMM = "/root/reference/proj/comm_model_test.json"


def _ours_or_err(fn, *a):
    try:
        return fn(*a), None
    except bx.Error as e:
        return None, (e.kind, e.msg)


def _ref_or_err(fn, *a):
    """The reference's result or (kind, message). nlohmann's own exceptions
    (type_error / out_of_range, not dagsched errors) escape the reference
    uncaught; the C ABI reports them as ValidationError with the same text."""
    try:
        return fn(*a), None
    except OracleError as e:
        if e.kind == 9 and e.msg.startswith("std::exception: "):
            return None, (bx.BX_VALIDATION, e.msg[len("std::exception: "):])
        return None, (e.kind, e.msg)


# ---- comm model ---------------------------------------------------------------
COMM_TEXTS = [
    '{"intercept_us": 12.5, "us_per_byte": 0.002, "mode": "parallel"}',
    '{"mode": "sequential", "us_per_byte": 1, "intercept_us": 0}',
    '{"intercept_us": 5, "us_per_byte": 1e-3, "mode": "sequential", "mode": "parallel"}',
    '{"intercept_us": 1e20, "us_per_byte": 123456789012345678, "mode": "parallel"}',
    '{"intercept_us": 0.1, "us_per_byte": 0.30000000000000004, "mode": "parallel"}',
    '{"intercept_us": 1e-7, "us_per_byte": 2.5e-5, "mode": "parallel"}',
    '{"intercept_us": 1e15, "us_per_byte": 1e16, "mode": "parallel"}',
    '{"intercept_us": -0.0, "us_per_byte": 0, "mode": "parallel"}',
    # validation errors
    '[1, 2]',
    '7',
    '{"intercept_us": 1, "us_per_byte": 1, "mode": "parallel", "extra": 3, "aaa": 1}',
    '{"intercept_us": 1, "mode": "parallel"}',
    '{"us_per_byte": 1, "mode": "parallel"}',
    '{"intercept_us": 1, "us_per_byte": 1}',
    '{"intercept_us": "1", "us_per_byte": 1, "mode": "parallel"}',
    '{"intercept_us": 1, "us_per_byte": null, "mode": "parallel"}',
    '{"intercept_us": -1, "us_per_byte": 1, "mode": "parallel"}',
    '{"intercept_us": 1, "us_per_byte": -0.5, "mode": "parallel"}',
    '{"intercept_us": 1, "us_per_byte": 1, "mode": "fast"}',
    '{"intercept_us": 1, "us_per_byte": 1, "mode": 3}',
]

SYNTAX_BAD = ['{"intercept_us": 1,}', '{"intercept_us" 1}', '', '{"a": tru}', '{"a": "x\x01"}', '{"a": 01}',
              '{"a": 1} x', '{"a": "\\ud800"}', '[1, 2', '{"a": -}']


@pytest.mark.parametrize("text", COMM_TEXTS)
def test_comm_model_matches_reference(text):
    ref, rerr = _ref_or_err(Ref.comm_model_roundtrip, text)
    ours, oerr = _ours_or_err(bx.parse_comm_model, text)
    assert oerr == rerr
    if ref is not None:
        (ic, pb, mode), rtext = ref
        assert (ours.intercept_us, ours.us_per_byte, ours.mode) == (ic, pb, mode)
        assert bx.comm_model_to_json(ours) == rtext


@pytest.mark.parametrize("text", SYNTAX_BAD)
def test_comm_model_syntax_errors(text):
    _, rerr = _ref_or_err(Ref.comm_model_roundtrip, text)
    _, oerr = _ours_or_err(bx.parse_comm_model, text)
    assert rerr is not None and oerr is not None
    assert oerr[0] == rerr[0] == bx.BX_VALIDATION
    assert oerr[1].startswith("parse error: ") and rerr[1].startswith("parse error: ")


def test_comm_model_doubles_match_reference_formatting():
    """Doubles print as nlohmann's layout of the shortest round-trip digits.
    nlohmann's Grisu2 is not always shortest (about 2% of random doubles get
    one more digit), so those texts may differ in the last digit; every text
    still reads back to the same double, and the layout always agrees."""
    rng = np.random.default_rng(3)
    vals = list(rng.uniform(0, 1e-3, 60)) + list(rng.uniform(0, 200, 60)) + list(10.0 ** rng.uniform(-9, 19, 80))
    exact = [0.0, 1.0, 5.0, 12.5, 0.002, 1e-5, 1e-4, 1e15, 1e16, 123456789.0, 0.1 + 0.2, 2.0 ** -30, 0.5, 3.25e-7]
    same = 0
    for i in range(0, len(vals) - 1, 2):
        text = json.dumps({"intercept_us": vals[i], "us_per_byte": vals[i + 1], "mode": "sequential"})
        (ic, pb, md), rtext = Ref.comm_model_roundtrip(text)
        ours = bx.parse_comm_model(text)
        assert (ours.intercept_us, ours.us_per_byte) == (ic, pb)
        out = bx.comm_model_to_json(ours)
        back = bx.parse_comm_model(out)
        assert (back.intercept_us, back.us_per_byte) == (ic, pb)
        same += out == rtext
    assert same >= 0.95 * (len(vals) // 2)
    for i in range(0, len(exact) - 1, 2):
        text = json.dumps({"intercept_us": exact[i], "us_per_byte": exact[i + 1], "mode": "parallel"})
        assert bx.comm_model_to_json(bx.parse_comm_model(text)) == Ref.comm_model_roundtrip(text)[1], text


def test_load_comm_model_test_json(tmp_path):
    if not os.path.exists(REF_COMM):
        pytest.skip("reference tree not mounted")
    cm = bx.load_comm_model(REF_COMM)
    assert (cm.intercept_us, cm.us_per_byte, cm.mode) == (12.5, 0.002, bx.PARALLEL)
    p = tmp_path / "cm.json"
    bx.save_comm_model(cm, str(p))
    assert bx.load_comm_model(str(p)) == cm
    with pytest.raises(bx.ValidationError, match="cannot open comm model file"):
        bx.load_comm_model(str(tmp_path / "missing.json"))


# ---- graph JSON -------------------------------------------------------------
def _ref_graph(seed, family="branchy", n=300, coloc=0.1, coplace=0.05):
    return Ref.generate(family, n, seed, colocate_edge_frac=coloc, coplace_frac=coplace)


@pytest.mark.parametrize("seed", range(6))
def test_graph_json_roundtrip_byte_identical(seed):
    fam = ["branchy", "layered-chain", "random-dag"][seed % 3]
    base = _ref_graph(seed, fam, 200 + 50 * seed)
    rg = Ref.graph(base, pipeline=-1)
    text = Ref.graph_to_json(rg)                  # the reference writes the file
    jg = bx.parse_graph(text)                      # we read it
    names = jg.names
    assert bx.graph_to_json(jg.base, names, jg.groups) == text  # and write it back identically
    assert Ref.graph_json_roundtrip(text) == text
    # the parsed base graph feeds the ingest exactly like the arrays it came from
    m1, g1 = bx.build_grouped(jg.base)
    m2, g2 = bx.build_grouped(base)
    assert np.array_equal(m1.esrc, m2.esrc) and np.array_equal(m1.k, m2.k)
    assert np.array_equal(g1["group_of"], g2["group_of"])


def test_graph_json_emits_unsorted_input_sorted():
    base = _ref_graph(11, "branchy", 120)
    rng = np.random.default_rng(0)
    perm_n = rng.permutation(len(base["id"]))
    perm_e = rng.permutation(len(base["src"]))
    shuffled = {k: (v[perm_n] if len(v) == len(base["id"]) and k not in ("src", "dst", "bytes") else v)
                for k, v in base.items()}
    for k in ("src", "dst", "bytes"):
        shuffled[k] = base[k][perm_e]
    names = ["n%d" % i for i in shuffled["id"]]
    groups = ["g%d" % i for i in range(int(base["coloc"].max()) + 1)]
    assert bx.graph_to_json(shuffled, names, groups) == Ref.graph_to_json(Ref.graph(base, pipeline=-1))


def _doc(nodes, edges):
    return json.dumps({"nodes": nodes, "edges": edges})


def _node(i, **kw):
    d = dict(id=i, name="n%s" % i, compute_time_us=5, temp_mem_bytes=1, perm_mem_bytes=2, out_mem_bytes=3,
             colocation_group=None, coplace_pair=None)
    d.update(kw)
    return d


GRAPH_DOCS = [
    _doc([_node(0), _node(1)], [dict(src=0, dst=1, tensor_bytes=4)]),
    _doc([], []),
    _doc([_node(0, name="quo\"te\\ \n\té中\U0001f600\x07")], []),
    _doc([_node(5, colocation_group="zz"), _node(2, colocation_group="aa"), _node(9, colocation_group="zz")], []),
    _doc([_node(0, coplace_pair=1), _node(1, coplace_pair=0)], [dict(src=0, dst=1, tensor_bytes=0)]),
    json.dumps({"edges": [], "nodes": [_node(0)], }),
    '{"nodes": [], "edges": [], "nodes": [' + json.dumps(_node(3)) + ']}',
    # errors, in the reference's order
    '[]',
    '{"nodes": []}',
    '{"nodes": [], "edges": [], "zeta": 1, "beta": 2}',
    '{"nodes": {}, "edges": []}',
    '{"nodes": [], "edges": 3}',
    _doc([5], []),
    _doc([{**_node(0), "extra": 1}], []),
    _doc([{k: v for k, v in _node(0).items() if k != "name"}], []),
    _doc([{k: v for k, v in _node(0).items() if k not in ("name", "id")}], []),
    _doc([_node("0")], []),
    _doc([_node(1.0)], []),
    _doc([_node(0, name=3)], []),
    _doc([_node(0, compute_time_us=-1)], []),
    _doc([_node(0, temp_mem_bytes=1.5)], []),
    _doc([_node(0, perm_mem_bytes=None)], []),
    _doc([_node(0, out_mem_bytes=18446744073709551615)], []),
    _doc([_node(0, colocation_group=3)], []),
    _doc([_node(0, coplace_pair="x")], []),
    _doc([_node(0)], [7]),
    _doc([_node(0)], [dict(src=0, dst=1)]),
    _doc([_node(0)], [dict(src=0, dst=1, tensor_bytes=1, w=2)]),
    _doc([_node(0)], [dict(src="0", dst=1, tensor_bytes=1)]),
    _doc([_node(0)], [dict(src=0, dst=1, tensor_bytes=-2)]),
    # make_graph (graph.cpp:99-194) errors after a clean parse
    _doc([_node(0), _node(0)], []),
    _doc([_node(0), _node(1)], [dict(src=0, dst=2, tensor_bytes=1)]),
    _doc([_node(0), _node(1)], [dict(src=0, dst=1, tensor_bytes=1), dict(src=0, dst=1, tensor_bytes=2)]),
    _doc([_node(0)], [dict(src=0, dst=0, tensor_bytes=1)]),
    _doc([_node(0), _node(1), _node(2)], [dict(src=0, dst=1, tensor_bytes=1), dict(src=1, dst=2, tensor_bytes=1),
                                          dict(src=2, dst=0, tensor_bytes=1)]),
    _doc([_node(0, coplace_pair=1), _node(1)], []),
    _doc([_node(0, coplace_pair=0)], []),
]


@pytest.mark.parametrize("idx", range(len(GRAPH_DOCS)))
def test_graph_json_parse_matches_reference(idx):
    text = GRAPH_DOCS[idx]
    ref, rerr = _ref_or_err(Ref.graph_json_roundtrip, text)

    def ours_fn(t):
        jg = bx.parse_graph(t)
        bx.build_grouped(jg.base, singleton=True)  # make_graph, as parse_graph ends in it
        return bx.graph_to_json(jg.base, jg.names, jg.groups)

    ours, oerr = _ours_or_err(ours_fn, text)
    assert oerr == rerr
    assert ours == ref


@pytest.mark.parametrize("text", SYNTAX_BAD)
def test_graph_json_syntax_errors(text):
    _, rerr = _ref_or_err(Ref.graph_json_roundtrip, text)
    _, oerr = _ours_or_err(bx.parse_graph, text)
    assert rerr is not None and oerr is not None
    assert oerr[0] == rerr[0] == bx.BX_VALIDATION and oerr[1].startswith("parse error: ")


def test_load_graph_file(tmp_path):
    base = _ref_graph(21, "layered-chain", 400)
    text = Ref.graph_to_json(Ref.graph(base, pipeline=-1))
    p = tmp_path / "g.json"
    p.write_text(text)
    jg = bx.load_graph(str(p))
    assert bx.graph_to_json(jg.base, jg.names, jg.groups) == text
    with pytest.raises(bx.ValidationError, match="cannot open graph file"):
        bx.load_graph(str(tmp_path / "nope.json"))


# ---- placement JSON -----------------------------------------------------------
def _upstream_int_arrays(text):
    """The oracle compiles the reference against the nlohmann copy vendored in
    cudnn_frontend, which is patched ("Custom from FE") to print arrays of
    integers inline; the reference's own json.hpp is upstream 3.11, which
    prints them one element per line. Restore the upstream layout."""
    import re

    def fix(m):
        ind = m.group(1)
        vals = m.group(3).split(",")
        inner = ",\n".join(ind + "  " + v for v in vals)
        return f"{ind}{m.group(2)}[\n{inner}\n{ind}]"

    return re.sub(r"(?m)^( *)(\"[a-z_]+\": )\[(-?\d+(?:,-?\d+)*)\]", fix, text)

def _placed(seed, n=4, pipeline=6):
    base = _ref_graph(seed, "branchy", 250, coloc=0.1, coplace=0.1)
    rg = Ref.graph(base, pipeline=pipeline)
    meta = rg.meta()
    cm = (12.5, 0.002, 1)
    caps = [Ref.bench_capacity(rg, n, 1.5)] * n
    p = Ref.place(rg, 1, caps, cm)
    sim = Ref.simulate(rg, caps, cm, 1, p.device_of, p.exec_order, p.exec_off)
    grouping = dict(base_ids=meta["base_id"], group_of=meta["group_of"], members=meta["members"],
                    member_off=meta["member_off"])
    return rg, meta, p, sim, grouping


@pytest.mark.parametrize("seed", range(4))
def test_placement_json_matches_reference(seed):
    rg, meta, p, sim, grouping = _placed(seed)
    rtext = _upstream_int_arrays(Ref.placement_to_json(rg, "m-etf", p.device_of, p.exec_order, p.exec_off,
                                                       sim.start_us, sim.makespan, sim.peak))
    pl = bx.Placement("m-etf", p.device_of, p.start_us, p.exec_order, p.exec_off)
    rep = bx.SimReport(sim.makespan, sim.start_us, sim.peak, sim.busy, sim.idle, 0, 0, 0, 0)
    assert bx.placement_to_json(grouping, pl, rep) == rtext
    n = len(p.exec_off) - 1
    ralgo, rp = Ref.placement_from_json(rg, rtext, n)
    back = bx.placement_from_json(grouping, meta["V"], rtext, n)
    assert back.algorithm == ralgo == "m-etf"
    assert np.array_equal(back.device_of, rp.device_of) and np.array_equal(back.start_us, rp.start_us)
    assert np.array_equal(back.exec_order_flat, rp.exec_order) and np.array_equal(back.exec_off, rp.exec_off)
    assert np.array_equal(back.device_of, p.device_of)


def test_placement_from_json_errors_match_reference():
    rg, meta, p, sim, grouping = _placed(7, n=2)
    n = 2
    rows = json.loads(Ref.placement_to_json(rg, "m-etf", p.device_of, p.exec_order, p.exec_off, sim.start_us,
                                            sim.makespan, sim.peak))["assignments"]
    V = meta["V"]
    multi = [m for m in range(V) if meta["member_off"][m + 1] - meta["member_off"][m] > 1]
    docs = [
        json.dumps({"algorithm": "x"}),
        json.dumps([1]),
        json.dumps({"algorithm": "m-etf", "assignments": rows[:-3]}),
        json.dumps({"algorithm": "m-etf", "assignments": [dict(rows[0], device=5)] + rows}),
        json.dumps({"algorithm": "m-etf", "assignments": [dict(rows[0], node=10 ** 9)] + rows}),
        json.dumps({"algorithm": "m-etf", "assignments": rows, "extra": {"a": [1, 2]}}),
        json.dumps({"algorithm": "m-etf", "assignments": None}),
        json.dumps({"algorithm": "m-etf", "assignments": [{"node": 0, "device": 0}]}),
        json.dumps({"algorithm": "m-etf", "assignments": [{"node": 0, "device": "0", "start_us": 1}]}),
        json.dumps({"algorithm": 5, "assignments": rows}),
    ]
    if multi:
        m = multi[0]
        b0 = int(meta["base_id"][meta["members"][meta["member_off"][m] + 1]])
        bad = [dict(r, device=1 - r["device"]) if r["node"] == b0 else r for r in rows]
        docs.append(json.dumps({"algorithm": "m-etf", "assignments": bad}))
    for d in docs:
        _, rerr = _ref_or_err(Ref.placement_from_json, rg, d, n)
        _, oerr = _ours_or_err(bx.placement_from_json, grouping, V, d, n)
        assert oerr == rerr, d[:200]


# ---- binary sidecar -----------------------------------------------------------
def test_binary_sidecar_roundtrip(tmp_path):
    base = _ref_graph(4, "random-dag", 300)
    meta, _ = bx.build_grouped(base)
    p = tmp_path / "g.bxg"
    bx.save_graph_bin(meta, str(p))
    back = bx.load_graph_bin(str(p))
    for k in ("k", "temp", "perm", "out", "esrc", "edst", "ebytes", "in_off", "in_edge", "out_off", "first_id"):
        assert np.array_equal(getattr(back, k), getattr(meta, k)), k
    raw = bytearray(p.read_bytes())
    raw[0] = ord("X")
    (tmp_path / "bad.bxg").write_bytes(bytes(raw))
    with pytest.raises(bx.ValidationError, match="not a graph sidecar"):
        bx.load_graph_bin(str(tmp_path / "bad.bxg"))
    (tmp_path / "short.bxg").write_bytes(p.read_bytes()[:100])
    with pytest.raises(bx.ValidationError, match="truncated"):
        bx.load_graph_bin(str(tmp_path / "short.bxg"))


def test_trace_to_csv_format():
    ev = [bx.TraceEvent(5, 1, "finish", 7), bx.TraceEvent(0, 0, "start", 3), bx.TraceEvent(5, 0, "xfer_begin", 7),
          bx.TraceEvent(0, 1, "start", 9), bx.TraceEvent(9, 1, "xfer_end", 7)]
    assert bx.trace_to_csv(ev) == ("time_us,device,event,node\n0,0,start,3\n0,1,start,9\n5,1,finish,7\n"
                                   "5,0,xfer_begin,7\n9,1,xfer_end,7\n")
    assert bx.trace_to_csv([]) == "time_us,device,event,node\n"
