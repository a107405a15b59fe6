"""Known-answer tests restated from the reference's own doctest suite.

Each KAT is data: a small graph, a roster, a comm model, the call, and the
expected outcome quoted from the reference test it restates. The same table
pins the CPU oracle (tests/test_oracle.py) and checks the CUDA path
(tests/test_gpu_parity.py).
"""
from __future__ import annotations

import numpy as np

SEQ, PAR = 0, 1
NO_COMM = (0.0, 0.0, SEQ)  # zero_comm_model(CommMode::Sequential), test_placers.cpp:17


def graph(nodes, edges):
    """nodes: (id, k, temp, perm, out); edges: (src_id, dst_id, bytes).
    Returns the singleton meta graph (make_graph sorts nodes by id and
    edges by (src, dst); transforms.cpp:300-327)."""
    nodes = sorted(nodes)
    idx = {n[0]: i for i, n in enumerate(nodes)}
    es = sorted((idx[s], idx[d], b) for s, d, b in edges)
    return dict(V=len(nodes), E=len(es),
                k=np.array([n[1] for n in nodes], np.int64),
                temp=np.array([n[2] for n in nodes], np.int64),
                perm=np.array([n[3] for n in nodes], np.int64),
                out=np.array([n[4] for n in nodes], np.int64),
                esrc=np.array([e[0] for e in es], np.int32),
                edst=np.array([e[1] for e in es], np.int32),
                ebytes=np.array([e[2] for e in es], np.int64),
                first_id=np.array([n[0] for n in nodes], np.int64))


def node(i, k, temp=0, perm=0, out=0):
    return (i, k, temp, perm, out)


def diamond(k=2, tensor=0, perm=0):  # test_util.hpp:31-37
    return graph([node(i, k, 0, perm) for i in range(4)],
                 [(0, 1, tensor), (0, 2, tensor), (1, 3, tensor), (2, 3, tensor)])


def chain(length, k=5, tensor=0):  # test_util.hpp:39-45
    return graph([node(i, k) for i in range(length)], [(i, i + 1, tensor) for i in range(length - 1)])


def manual(device_of, n):
    """test_simulator.cpp `manual`: exec lists in ascending node order."""
    dev = np.array(device_of, np.int32)
    order, off = [], [0]
    for d in range(n):
        order += [j for j in range(len(dev)) if dev[j] == d]
        off.append(len(order))
    return dev, np.array(order, np.int32), np.array(off, np.int32)


# ---- placer KATs (proj/tests/test_placers.cpp) -----------------------------
# (name, graph, algo, caps, cm, fav_child, check(placement, stats) | ("raise", kind, substring))
def placer_kats():
    um = diamond(2, 0, 1)  # unit_mem_diamond, test_placers.cpp:19-21
    k = []
    k.append(("mtopo_fill_cap3", um, 0, [100, 100], NO_COMM, None,  # :25-32
              lambda p, s: (p.device_of.tolist() == [0, 0, 0, 1]
                            and p.exec_lists() == [[0, 1, 2], [3]])))
    k.append(("mtopo_single_device", um, 0, [100], NO_COMM, None,  # :34-38
              lambda p, s: p.device_of.tolist() == [0, 0, 0, 0]))
    g = graph([node(0, 1, 0, 5, 0), node(1, 1, 0, 1, 0), node(2, 1, 0, 1, 0), node(3, 1, 0, 1, 0)],
              [(0, 1, 0), (1, 2, 0), (2, 3, 0)])
    k.append(("mtopo_cap_exceeds", g, 0, [8, 8], NO_COMM, None, ("raise", 3, "m-etf")))  # :40-50
    g = graph([node(0, 10), node(1, 10)], [])
    k.append(("metf_spreads_independent", g, 1, [1000, 1000], NO_COMM, None,  # :81-87
              lambda p, s: p.start_us.tolist() == [0, 0] and p.device_of[0] != p.device_of[1]))
    g = graph([node(0, 4), node(1, 1)], [(0, 1, 1000)])
    k.append(("metf_colocates_chain", g, 1, [1000, 1000], (0.0, 1.0, SEQ), None,  # :89-97
              lambda p, s: p.device_of[0] == p.device_of[1] and p.start_us[1] == 4))
    k.append(("metf_discards_full_devices", um, 1, [2, 2], NO_COMM, None,  # :99-111
              lambda p, s: [len(x) for x in p.exec_lists()] == [2, 2] and s[0] > 0))
    g = graph([node(0, 1, 0, 50, 0)], [])
    k.append(("metf_fits_nowhere", g, 1, [10, 10], NO_COMM, None, ("raise", 3, "fits on no device")))  # :113-117
    g = graph([node(0, 4), node(1, 2)], [(0, 1, 3)])
    k.append(("msct_keeps_favorite", g, 2, [1000, 1000], (0.0, 1.0, SEQ), [1, -1],  # :153-164
              lambda p, s: p.device_of[0] == p.device_of[1] and p.start_us[1] == 4))
    g = graph([node(0, 10), node(1, 6), node(2, 2)], [(0, 1, 1), (0, 2, 8)])
    k.append(("msct_awake_reservation", g, 2, [1000, 1000], (0.0, 1.0, PAR), [2, -1, -1],  # :166-188
              lambda p, s: s[2] > 0 and p.device_of[2] == p.device_of[0] and p.start_us[2] == 10))
    k.append(("metf_no_reservation", g, 1, [1000, 1000], (0.0, 1.0, PAR), None,  # :187
              lambda p, s: p.start_us[2] > 10))
    # roster validation (placers.cpp:19-29)
    k.append(("roster_nonpositive", um, 1, [0, 5], NO_COMM, None, ("raise", 2, "capacities must be positive")))
    k.append(("fav_size_mismatch", um, 2, [100, 100], NO_COMM, [1, -1], ("raise", 2, "favorite map")))
    # acyclicity (meta_topo_order) on a hand-built cyclic meta graph
    cyc = graph([node(0, 1), node(1, 1), node(2, 1)], [(0, 1, 0), (1, 2, 0), (2, 1, 0)])
    k.append(("cyclic_meta_graph", cyc, 1, [100], NO_COMM, None, ("raise", 2, "meta graph is cyclic; groups of base node ids {1, 2} remain")))
    return k


# ---- simulator KATs (proj/tests/test_simulator.cpp) -------------------------
# (name, graph, device_of, n, caps, cm, mem_mode, check(report) | ("raise", kind, substring))
TP, GS = 1, 0


def simulator_kats():
    k = []
    g = graph([node(0, 10, 3, 5, 7)], [])
    k.append(("single_node", g, [0], 1, [100], (0.0, 0.0, PAR), TP,  # :30-40
              lambda r: (r.makespan, r.peak[0], r.transfer_count, r.busy[0], r.idle[0]) == (10, 15, 0, 10, 0)))
    g = graph([node(0, 3), node(1, 5)], [(0, 1, 2)])
    k.append(("cross_device_chain", g, [0, 1], 2, [100, 100], (0.0, 1.0, SEQ), TP,  # :42-53
              lambda r: (r.makespan, r.transfer_count, r.transfer_bytes, r.start_us[1]) == (10, 1, 2, 5)))
    g = graph([node(0, 2), node(1, 2), node(2, 2)], [(0, 1, 4), (0, 2, 4)])
    k.append(("shared_transfer", g, [0, 1, 1], 2, [100, 100], (0.0, 1.0, SEQ), TP,  # :55-67
              lambda r: (r.transfer_count, r.duplicate_transfers, r.cache_hits) == (1, 0, 1)))
    g = graph([node(0, 5, 0, 0, 60), node(1, 5, 0, 0, 60)], [(0, 1, 0)])
    k.append(("memory_violation_t5", g, [0, 0], 1, [100], (0.0, 0.0, PAR), TP, ("raise", 3, "t=5")))  # :69-83
    g = graph([node(0, 5, 0, 0, 60), node(1, 5, 0, 0, 60), node(2, 5, 0, 0, 60)], [(0, 1, 0), (1, 2, 0)])
    k.append(("graph_static_frees", g, [0, 0, 0], 1, [150], (0.0, 0.0, PAR), GS,  # :85-103
              lambda r: (r.peak[0], r.makespan) == (120, 15)))
    k.append(("persistent_overflows", g, [0, 0, 0], 1, [150], (0.0, 0.0, PAR), TP, ("raise", 3, "memory violation")))
    g = graph([node(0, 5, 60, 0, 0), node(1, 5, 60, 0, 0)], [])
    k.append(("release_before_reserve", g, [0, 0], 1, [100], (0.0, 0.0, PAR), TP,  # :116-127
              lambda r: r.peak[0] == 60 and r.makespan == 10))
    c6 = chain(6, 7)
    k.append(("six_chain_42", c6, [0] * 6, 1, [100], (0.0, 0.0, PAR), TP, lambda r: r.makespan == 42))
    return k


DEADLOCK = graph([node(0, 5), node(1, 5)], [(0, 1, 0)])  # test_simulator.cpp:105-114


# ---- comm_time KATs (proj/tests/test_cost_model.cpp:13-19) -----------------
COMM_KATS = [((100.0, 0.01), 0, 100), ((100.0, 0.01), 10_000, 200), ((0.0, 0.0), 123, 0), ((0.0, 0.05), 10, 1)]
