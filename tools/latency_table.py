"""Single-graph placement latency: GPU (device-resident, CUDA events around
the placer kernel) vs the compiled reference (one host core, run_placer's
scope), with a bit-exact check of the two placements.

python tools/latency_table.py [names...]      (default: the standard set)
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

CASES = {
    "layered100k_x4": (lambda: W.layered_dag_fast(100, 1000, 3), 4, "m-etf", 1.2),
    "layered100k_x8": (lambda: W.layered_dag_fast(100, 1000, 3), 8, "m-etf", 1.2),
    "layered100k_x64": (lambda: W.layered_dag_fast(100, 1000, 3), 64, "m-etf", 1.2),
    "grid100k_x8": (lambda: W.grid_chain(6250, 16, 4), 8, "m-etf", 1.2),
    "wide100k_x16": (lambda: W.wide_random(100000, 5), 16, "m-etf", 1.2),
    "layered100k_x4_sct": (lambda: W.layered_dag_fast(100, 1000, 3), 4, "m-sct", 1.2),
    "c4_layered1M_x64": (lambda: W.layered_dag_fast(1000, 1000, 1), 64, "m-etf", 1.5),
    "c4_layered1M_x64_tight": (lambda: W.layered_dag_fast(1000, 1000, 1), 64, "m-etf", 1.05),
    "c4_layered1M_x64_sct": (lambda: W.layered_dag_fast(1000, 1000, 1), 64, "m-sct", 1.5),
    # the reference's own layered-chain family (generate_graph, 4 stacked chains,
    # seed 55; SURVEY Appendix A / BASELINE.md §2): a 4-wide frontier
    "refchain100k_x4": (lambda: _refchain(100000), 4, "m-etf", 1.5),
    "refchain100k_x8": (lambda: _refchain(100000), 8, "m-etf", 1.5),
    "seq_refchain100k_x4": (lambda: _refchain(100000), 4, "m-etf", 1.5),
    "seq_refchain100k_x8": (lambda: _refchain(100000), 8, "m-etf", 1.5),
    "refchain1M_x64": (lambda: _refchain(1000000), 64, "m-etf", 1.5),
    "refchain100k_x8_sct": (lambda: _refchain(100000), 8, "m-sct", 1.5),
    "refchain100k_x4_sct": (lambda: _refchain(100000), 4, "m-sct", 1.5),
    "seq_refchain100k_x4_sct": (lambda: _refchain(100000), 4, "m-sct", 1.5),
    # sequential comm mode (queues on both endpoints), the survey probe's model {5 us, 0.001 us/B}
    "seq_layered100k_x4": (lambda: W.layered_dag_fast(100, 1000, 3), 4, "m-etf", 1.2),
    "seq_layered100k_x8": (lambda: W.layered_dag_fast(100, 1000, 3), 8, "m-etf", 1.2),
    "seq_wide100k_x16": (lambda: W.wide_random(100000, 5), 16, "m-etf", 1.2),
}
COMM_SEQ = (5.0, 0.001, 0)


def _refchain(V, layers=4, seed=55):
    """generate_graph(layered-chain) from the compiled reference (input
    generation only), as a singleton meta-graph dict."""
    from oracle import Ref
    base = Ref.generate("layered-chain", V, seed, layers=layers)
    ids = base["id"]
    order = np.argsort(ids, kind="stable")
    idx = np.empty_like(order)
    idx[order] = np.arange(len(ids))
    src = idx[order[np.searchsorted(ids[order], base["src"])]]  # node id -> make_graph index
    dst = idx[order[np.searchsorted(ids[order], base["dst"])]]
    e = np.lexsort((dst, src))
    return dict(V=len(ids), k=base["k"][order], temp=base["temp"][order], perm=base["perm"][order],
                out=base["out"][order], esrc=src[e].astype(np.int32), edst=dst[e].astype(np.int32),
                ebytes=base["bytes"][e], name="refchain")


def run_config(name, cpu=True, reps=10):
    """BASELINE configs C1-C3: our ingest + GPU placer vs the reference's
    transforms + placer (one core), same base graph. GPU: placer kernels on
    device-resident inputs (CUDA events, median of `reps` after a warm-up)
    and the one-shot drop-in call bx_place end to end (host arrays in and
    out, median of `reps`); CPU: the reference place_* on one core, median of
    `reps` back-to-back calls (run_placer's scope)."""
    import statistics
    import time as _t
    gen, n, algos, kw, f = W.CONFIGS[name]
    g = gen()
    t0 = _t.perf_counter()
    meta, _ = bx.build_grouped(g, **kw)
    ingest_ms = (_t.perf_counter() - t0) * 1e3
    cap = W.meta_capacity(meta, n, f)
    cm = bx.CommModel(*W.COMM_TEST)
    rows = []
    for algo in algos:
        fav = fav_first(meta.esrc, meta.edst, meta.V) if algo == "m-sct" else None
        plan = bx.Plan([meta], [bx.Job(0, algo, np.full(n, cap, np.int64), cm, fav)])
        plan.upload()
        plan.place()
        for _ in range(reps):
            plan.place()
        ms = plan.kernel_times(reps)
        plan.download()
        st, msg = plan.status(0)
        p = plan.result(0) if st == 0 else None
        kern = plan.job_kernel(0)
        plan.close()
        caps = np.full(n, cap, np.int64)
        one = []
        for _ in range(reps + 1):
            t1 = _t.perf_counter()
            q = bx._one(meta, algo, caps, cm, fav)
            one.append((_t.perf_counter() - t1) * 1e3)
        row = {"case": name, "algo": algo, "base_V": g["V"], "meta_V": meta.V, "meta_E": meta.E, "n": n,
               "ingest_ms_host": round(ingest_ms, 2), "gpu_kernel_ms": statistics.median(ms), "kernel": kern,
               "gpu_oneshot_ms": statistics.median(one[1:]), "status": st}
        if cpu:
            from oracle import Ref
            pipe = (2 if kw.get("coplacement", True) else 0) | (4 if kw.get("fusion", True) else 0)
            rg = Ref.graph(g, pipe)
            code = {"m-topo": 0, "m-etf": 1, "m-sct": 2}[algo]
            o = Ref.place(rg, code, [cap] * n, W.COMM_TEST, fav)
            walls = Ref.place_timed(rg, code, [cap] * n, W.COMM_TEST, reps, fav)
            row["cpu_ref_ms"] = float(np.median(walls)) / 1e6
            row["cpu_ref_runs"] = reps
            row["bit_exact"] = bool(p is not None and np.array_equal(o.device_of, p.device_of)
                                    and np.array_equal(o.start_us, p.start_us)
                                    and np.array_equal(o.exec_order, p.exec_order_flat)
                                    and np.array_equal(o.exec_off, p.exec_off)
                                    and (algo == "m-topo" or tuple(o.stats) == tuple(p.stats))
                                    and q == p)
            row["speedup"] = row["cpu_ref_ms"] / row["gpu_kernel_ms"]
            row["speedup_oneshot"] = row["cpu_ref_ms"] / row["gpu_oneshot_ms"]
        rows.append(row)
    return rows


def fav_first(esrc, edst, V):
    fav = np.full(V, -1, np.int32)
    claimed = np.zeros(V, bool)
    for s, d in zip(esrc.tolist(), edst.tolist()):
        if fav[s] < 0 and not claimed[d]:
            fav[s] = d
            claimed[d] = True
    return fav


def run(name, cpu=True, reps=3):
    mk, n, algo, f = CASES[name]
    g = mk()
    m = W.as_meta_dict(g)
    gg = bx.MetaGraph.from_dict(m)
    cmt = COMM_SEQ if name.startswith("seq_") else W.COMM_TEST
    cm = bx.CommModel(*cmt)
    caps = np.full(n, W.bench_capacity(g, n, f), np.int64)
    fav = fav_first(g["esrc"], g["edst"], g["V"]) if algo == "m-sct" else None
    plan = bx.Plan([gg], [bx.Job(0, algo, caps, cm, fav)])
    plan.upload()
    ms = []
    for _ in range(reps + 1):
        plan.place()
        ms.append(plan.kernel_ms())
    plan.download()
    p = plan.result(0)
    row = {"case": name, "V": gg.V, "E": gg.E, "n": n, "algo": algo, "gpu_kernel_ms": min(ms[1:]),
           "gpu_ms_all": [round(x, 2) for x in ms[1:]]}
    if cpu:
        from oracle import Ref
        rg = Ref.graph(W.as_ref_base(g), -1)
        t0 = time.time()
        o = Ref.place(rg, 2 if algo == "m-sct" else 1, caps, cmt, fav)
        row["cpu_ref_ms"] = o.wall_ns / 1e6
        row["cpu_wall_s"] = round(time.time() - t0, 2)
        row["bit_exact"] = bool(np.array_equal(o.device_of, p.device_of) and np.array_equal(o.start_us, p.start_us)
                                and np.array_equal(o.exec_order, p.exec_order_flat))
        row["speedup"] = row["cpu_ref_ms"] / row["gpu_kernel_ms"]
    plan.close()
    return row


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or list(CASES)
    cpu = "--no-cpu" not in sys.argv
    for nm in names:
        if nm in W.CONFIGS:
            for r in run_config(nm, cpu=cpu):
                print(json.dumps(r), flush=True)
        else:
            print(json.dumps(run(nm, cpu=cpu)), flush=True)
