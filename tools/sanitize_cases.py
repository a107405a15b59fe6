"""Small inputs through every kernel of the engine, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck). Each case is also checked
against the C restatement, so a sanitizer run is a parity run too.

compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from oracle import Restate  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

ALGO = ["m-topo", "m-etf", "m-sct"]
KERNELS = {
    "small-frontier": {},
    "warp": {"wide_min_vn": (1 << 31) - 1, "no_small_frontier": 1},
    "rounds": {"wide_min_vn": 0, "no_small_frontier": 1},
    "rounds16": {"wide_min_vn": 0, "no_small_frontier": 1, "list_len": 16},
}


def fav_first(m):
    fav = np.full(m["V"], -1, np.int32)
    claimed = np.zeros(m["V"], bool)
    for s, d in zip(m["esrc"].tolist(), m["edst"].tolist()):
        if fav[s] < 0 and not claimed[d]:
            fav[s] = d
            claimed[d] = True
    return fav


def main():
    ran = {}
    for g in (W.branchy(3, 1), W.layered_dag(5, 8, 2), W.wide_random(60, 3)):
        m = W.as_meta_dict(g)
        gg = bx.MetaGraph.from_dict(m)
        fav = fav_first(m)
        for n in (2, 5):
            caps = [W.bench_capacity(g, n, 1.3)] * n
            for cmv in ((12.5, 0.002, 1), (5.0, 0.001, 0)):
                cm = bx.CommModel(*cmv)
                for kname, opts in KERNELS.items():
                    for algo in (0, 1, 2):
                        fv = fav if algo == 2 else None
                        plan = bx.Plan([gg], [bx.Job(0, ALGO[algo], np.array(caps, np.int64), cm, fv)], options=opts)
                        plan.upload()
                        plan.place()
                        plan.download()
                        kern = plan.job_kernel(0)
                        ran[kern] = ran.get(kern, 0) + 1
                        p = plan.result(0)
                        o = Restate.place(m, algo, caps, cmv, fv)
                        assert np.array_equal(p.device_of, o.device_of) and np.array_equal(p.start_us, o.start_us)
                        for mem in (0, 1):  # K4f (parallel comm) and K4 (sequential comm)
                            plan.simulate(mem)
                            r = plan.sim_download()[0]
                            s = Restate.simulate(m, caps, cmv, mem, o.device_of, o.exec_order, o.exec_off)
                            assert r.makespan_us == s.makespan
                        plan.close()
                rep = bx.simulate(gg, p, caps, cm, 1, record_trace=True)
                assert rep.trace
        # K3, schedulable_time, critical_path_us
        x = np.random.default_rng(1).random(m["E"])
        bx.round_and_extract(m["V"], m["esrc"], m["edst"], x, 0.3)
        st = bx.PlacerState(m["V"], 3, bx.PARALLEL)
        bx.schedulable_times(st, list(range(m["V"])), [0] * m["V"], gg, bx.CommModel(12.5, 0.002, 1))
        bx.critical_path_us(gg)
    # m-TOPO single pops and the acyclicity check's level-peel fallback
    # (a randomly renumbered DAG), and its cycle residue (one back edge)
    g = W.as_meta_dict(W.layered_dag(30, 10, 4))
    perm = np.random.default_rng(2).permutation(g["V"])
    r = dict(V=g["V"])
    for f in ("k", "temp", "perm", "out"):
        a = np.empty_like(g[f])
        a[perm] = g[f]
        r[f] = a
    sv, dv = perm[g["esrc"]], perm[g["edst"]]
    o = np.lexsort((dv, sv))
    r.update(esrc=sv[o].astype(np.int32), edst=dv[o].astype(np.int32), ebytes=np.asarray(g["ebytes"])[o], E=len(o))
    gg = bx.MetaGraph.from_dict(r)
    caps = [10 ** 12] * 3
    for algo in (0, 1):
        p = bx._one(gg, ALGO[algo], caps, bx.CommModel(12.5, 0.002, 1))
        o = Restate.place(r, algo, caps, (12.5, 0.002, 1))
        assert np.array_equal(p.device_of, o.device_of) and np.array_equal(p.start_us, o.start_us)
    x = int(g["esrc"][0])  # follow first out-edges to a sink: a path, so sink -> start closes a cycle
    start = x
    while True:
        nxt = g["edst"][g["esrc"] == x]
        if len(nxt) == 0:
            break
        x = int(nxt[0])
    last, first = int(perm[x]), int(perm[start])
    cyc = dict(r, esrc=np.append(r["esrc"], last).astype(np.int32), edst=np.append(r["edst"], first).astype(np.int32),
               ebytes=np.append(r["ebytes"], 4096), E=r["E"] + 1)
    o = np.lexsort((cyc["edst"], cyc["esrc"]))
    cyc.update(esrc=cyc["esrc"][o], edst=cyc["edst"][o], ebytes=cyc["ebytes"][o])
    try:
        bx._one(bx.MetaGraph.from_dict(cyc), "m-etf", caps, bx.CommModel(12.5, 0.002, 1))
    except bx.CycleError:
        ran["cycle"] = ran.get("cycle", 0) + 1
    # a batch: the many-job dispatch (warp kernel lists, the side stream)
    graphs = [W.branchy(3, s) for s in range(4)]
    mgs = [bx.MetaGraph.from_dict(W.as_meta_dict(g)) for g in graphs]
    jobs = [bx.Job(i % 4, "m-etf", np.full(n, W.bench_capacity(graphs[i % 4], n, 1.2), np.int64),
                   bx.CommModel(12.5, 0.002, i % 2)) for i, n in enumerate([2, 3, 4, 8] * 50)]
    plan = bx.Plan(mgs, jobs)
    plan.upload()
    plan.place()
    plan.download()
    assert all(plan.status(i)[0] == 0 for i in range(len(jobs)))
    plan.close()
    # a small LP (host IPM, GPU factorisation)
    gg = bx.MetaGraph.from_dict(W.as_meta_dict(W.branchy(2, 9)))
    bx.sct_favorites(gg, bx.CommModel(12.5, 0.002, 1))
    print("sanitize cases ok; kernels:", ran)


if __name__ == "__main__":
    main()
