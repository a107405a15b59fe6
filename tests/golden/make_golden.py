"""Generates tests/golden/placements.npz + index.json from the REFERENCE
ITSELF (oracle/_ref/libdagsched_ref.so = /root/reference/proj/src compiled
unmodified). Run in the container that mounts /root/reference:

    make -C oracle && python tests/golden/make_golden.py

Graphs come from the reference's own generator (generate_graph,
proj/src/generator.cpp:173) and from paper_2301_08695_b200.workloads; each
case stores the singleton meta graph, the job, and the reference's
Placement + PlacerStats (or error kind/message) and SimReport for both
memory modes.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import OracleError, Ref  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402


def fav_first(m):
    fav = np.full(m["V"], -1, np.int32)
    claimed = set()
    for e in range(m["E"]):
        s, d = int(m["esrc"][e]), int(m["edst"][e])
        if fav[s] < 0 and d not in claimed:
            fav[s] = d
            claimed.add(d)
    return fav


def main():
    arrays, index = {}, []
    graphs = []
    for seed, fam in [(3, "branchy"), (4, "layered-chain"), (5, "random-dag"), (11, "branchy"),
                      (12, "layered-chain"), (13, "random-dag")]:
        g = Ref.generate(fam, 120 + 15 * seed, seed, layers=6, edge_prob=0.04)
        graphs.append((f"ref-{fam}-{seed}", g))
    for name, g in [("wl-layered", W.layered_dag(12, 20, 5)), ("wl-grid", W.grid_chain(30, 8, 6)),
                    ("wl-branchy", W.branchy(10, 7)), ("wl-wide", W.wide_random(300, 8))]:
        graphs.append((name, W.as_ref_base(g)))
    case = 0
    for gname, base in graphs:
        rg = Ref.graph(base, -1)
        m = rg.meta()
        gi = len([k for k in arrays if k.startswith("g") and k.endswith("_k")])
        for f in ("k", "temp", "perm", "out", "esrc", "edst", "ebytes", "first_id"):
            arrays[f"g{gi}_{f}"] = m[f]
        fav = fav_first(m)
        for n, factors in ((2, (1.02, 2.0)), (4, (1.01, 1.2)), (8, (1.05,))):
            for fct in factors:
                cap = Ref.bench_capacity(rg, n, fct)
                for het in (False, True):
                    caps = [cap] * n if not het else [int(cap * (0.85 + 0.1 * d)) for d in range(n)]
                    for mode in (0, 1):
                        cm = (12.5, 0.002, mode) if mode else (5.0, 0.001, 0)
                        for algo in (0, 1, 2):
                            fv = fav if algo == 2 else None
                            rec = dict(case=case, graph=gi, gname=gname, n=n, caps=caps, cm=cm, algo=algo,
                                       fav=algo == 2)
                            try:
                                p = Ref.place(rg, algo, caps, cm, fv)
                                rec["status"] = 0
                                arrays[f"c{case}_device_of"] = p.device_of
                                arrays[f"c{case}_start"] = p.start_us
                                arrays[f"c{case}_exec_order"] = p.exec_order
                                arrays[f"c{case}_exec_off"] = p.exec_off
                                rec["stats"] = [int(x) for x in p.stats]
                                sims = []
                                for mm in (0, 1):
                                    try:
                                        r = Ref.simulate(rg, caps, cm, mm, p.device_of, p.exec_order,
                                                         p.exec_off)
                                        sims.append(dict(status=0, makespan=r.makespan,
                                                         peak=r.peak.tolist(), busy=r.busy.tolist(),
                                                         idle=r.idle.tolist(),
                                                         xfer=[r.transfer_count, r.transfer_bytes,
                                                               r.duplicate_transfers, r.cache_hits]))
                                        arrays[f"c{case}_sim{mm}_start"] = r.start_us
                                    except OracleError as e:
                                        sims.append(dict(status=e.kind, msg=e.msg))
                                rec["sims"] = sims
                            except OracleError as e:
                                rec["status"] = e.kind
                                rec["msg"] = e.msg
                            index.append(rec)
                            case += 1
    np.savez_compressed(os.path.join(HERE, "placements.npz"), **arrays)
    json.dump(index, open(os.path.join(HERE, "index.json"), "w"), indent=0)
    ok = sum(1 for r in index if r["status"] == 0)
    print(f"{len(index)} cases ({ok} placed, {len(index) - ok} errors), {len(graphs)} graphs")


if __name__ == "__main__" and "--ingest" not in sys.argv:
    main()


def make_ingest():
    """tests/golden/ingest.npz: reference transforms (colocation, co-placement,
    fusion) of seeded generator graphs with colocation groups and coplace pairs."""
    arrays, index = {}, []
    case = 0
    for seed, fam, cf, pf in [(21, "branchy", 0.2, 0.1), (22, "layered-chain", 0.1, 0.2),
                              (23, "random-dag", 0.3, 0.05), (24, "branchy", 0.0, 0.3)]:
        g = Ref.generate(fam, 220, seed, layers=5, edge_prob=0.04, colocate_edge_frac=cf, coplace_frac=pf)
        for pipe in (-1, 0, 2, 4, 6):
            try:
                r = Ref.graph(g, pipe).meta()
            except OracleError:
                continue
            for k in ("id", "k", "temp", "perm", "out", "coloc", "has_pair", "pair", "src", "dst", "bytes"):
                arrays[f"c{case}_in_{k}"] = g[k]
            for k in ("k", "temp", "perm", "out", "esrc", "edst", "ebytes", "group_of", "ecount", "member_off",
                      "members", "first_id"):
                arrays[f"c{case}_out_{k}"] = r[k]
            index.append(dict(case=case, pipe=pipe, family=fam, seed=seed, V=int(r["V"])))
            case += 1
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **arrays)
    json.dump(index, open(os.path.join(HERE, "ingest_index.json"), "w"), indent=0)
    print(f"{len(index)} ingest cases")


if __name__ == "__main__" and "--ingest" in sys.argv:
    make_ingest()
