"""Quick CUDA-vs-reference parity sweep (dev tool; the tests are in tests/)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2301_08695_b200 as bx
from oracle import Ref, Restate, OracleError

def fav_first(m):
    fav = np.full(m["V"], -1, np.int32); claimed = set()
    for e in range(m["E"]):
        s, d = int(m["esrc"][e]), int(m["edst"][e])
        if fav[s] < 0 and d not in claimed:
            fav[s] = d; claimed.add(d)
    return fav

ok = bad = 0
t0 = time.time()
for seed in range(1, int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    fam = ["branchy", "layered-chain", "random-dag"][seed % 3]
    g = Ref.generate(fam, 150 + 10 * seed, seed, layers=5, edge_prob=0.05)
    rg = Ref.graph(g, -1)
    m = rg.meta()
    gg = bx.MetaGraph.from_dict(m)
    for n in (2, 4, 8):
        for f in (1.01, 1.1, 2.0):
            cap = Ref.bench_capacity(rg, n, f)
            caps = [cap] * n
            if seed % 2: caps = [int(cap * (0.8 + 0.1 * d)) for d in range(n)]
            for mode in (0, 1):
                cm = (12.5, 0.002, mode)
                for algo in (0, 1, 2):
                    fav = fav_first(m) if algo == 2 else None
                    try:
                        a = Ref.place(rg, algo, caps, cm, fav); ea = None
                    except OracleError as e:
                        a = None; ea = (e.kind, e.msg)
                    try:
                        b = bx._one(gg, ["m-topo", "m-etf", "m-sct"][algo], caps, bx.CommModel(*cm), fav); eb = None
                    except bx.Error as e:
                        b = None; eb = (e.kind, e.msg)
                    if a is None or b is None:
                        if ea == eb: ok += 1
                        else:
                            bad += 1; print("ERR", seed, n, f, mode, algo, ea, eb)
                        continue
                    same = (np.array_equal(a.device_of, b.device_of) and np.array_equal(a.start_us, b.start_us)
                            and np.array_equal(a.exec_order, b.exec_order_flat) and np.array_equal(a.exec_off, b.exec_off)
                            and (algo == 0 or tuple(a.stats) == tuple(b.stats)))
                    if same:
                        ok += 1
                    else:
                        bad += 1
                        if bad < 10:
                            nd = int((a.device_of != b.device_of).sum()); ns = int((a.start_us != b.start_us).sum())
                            print("MISMATCH", seed, fam, n, f, mode, algo, "dev", nd, "start", ns, a.stats, b.stats)
                    # simulate both
                    if same and algo:
                        for mm in (0, 1):
                            try:
                                ra = Ref.simulate(rg, caps, cm, mm, a.device_of, a.exec_order, a.exec_off); sa = None
                            except OracleError as e:
                                ra = None; sa = (e.kind, e.msg)
                            try:
                                rb = bx.simulate(gg, b, caps, bx.CommModel(*cm), mm); sb = None
                            except bx.Error as e:
                                rb = None; sb = (e.kind, e.msg)
                            if ra is None or rb is None:
                                if sa != sb: bad += 1; print("SIMERR", sa, sb)
                                continue
                            if not (ra.makespan == rb.makespan_us and np.array_equal(ra.start_us, rb.start_us)
                                    and np.array_equal(ra.peak, rb.peak_bytes) and np.array_equal(ra.busy, rb.busy_us)
                                    and (ra.transfer_count, ra.transfer_bytes, ra.duplicate_transfers, ra.cache_hits)
                                    == (rb.transfer_count, rb.transfer_bytes, rb.duplicate_transfers, rb.cache_hits)):
                                bad += 1; print("SIMMISMATCH", seed, n, mode, mm, ra.makespan, rb.makespan_us)
print("ok", ok, "bad", bad, "secs", round(time.time() - t0, 1))
