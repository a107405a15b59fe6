"""Per-commit latency breakdown (clock64 phases) of the list placer on the
BASELINE configs and the 100k single-graph cases, for both the warp kernel and
the round kernel (forced through plan options).

python tools/config_profile.py [case ...]
"""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402
sys.path.insert(0, "tools")
from latency_table import fav_first  # noqa: E402


def cases():
    cm = bx.CommModel(*W.COMM_TEST)
    for name, (gen, n, algos, kw, f) in W.CONFIGS.items():
        g = gen()
        meta, _ = bx.build_grouped(g, **kw)
        cap = W.meta_capacity(meta, n, f)
        for algo in algos:
            if algo == "m-topo":
                continue
            fav = fav_first(meta.esrc, meta.edst, meta.V) if algo == "m-sct" else None
            yield name, meta, bx.Job(0, algo, np.full(n, cap, np.int64), cm, fav)
    for name, mk, n in (("grid100k_x8", lambda: W.grid_chain(6250, 16, 4), 8),
                        ("layered100k_x4", lambda: W.layered_dag_fast(100, 1000, 3), 4),
                        ("wide100k_x16", lambda: W.wide_random(100000, 5), 16),
                        ("layered100k_x64", lambda: W.layered_dag_fast(100, 1000, 3), 64),
                        ("layered100k_x16", lambda: W.layered_dag_fast(100, 1000, 3), 16),
                        ("layered30k_x64", lambda: W.layered_dag_fast(30, 1000, 3), 64)):
        g = mk()
        gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
        yield name, gg, bx.Job(0, "m-etf", np.full(n, W.bench_capacity(g, n, 1.2), np.int64), cm)
    cms = bx.CommModel(5.0, 0.001, 0)  # sequential comm (the survey probe's model)
    for name, mk, n in (("seq_layered100k_x8", lambda: W.layered_dag_fast(100, 1000, 3), 8),
                        ("seq_wide100k_x16", lambda: W.wide_random(100000, 5), 16),
                        ("seq_layered20k_x8", lambda: W.layered_dag_fast(20, 1000, 3), 8)):
        g = mk()
        gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
        yield name, gg, bx.Job(0, "m-etf", np.full(n, W.bench_capacity(g, n, 1.2), np.int64), cms)
    # the reference's own layered-chain graph (K2q in sequential comm)
    from latency_table import _refchain
    g = _refchain(100000)
    gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
    yield "seq_refchain100k_x4", gg, bx.Job(0, "m-etf", np.full(4, W.bench_capacity(g, 4, 1.5), np.int64), cms)


def main():
    want = set(a for a in sys.argv[1:])
    for name, gg, job in cases():
        if want and name not in want:
            continue
        kerns = os.environ.get("CP_KERNELS", "small,warp,rounds").split(",")
        # small: the small-frontier kernel (phases: argmin = keys + selection,
        # commit = cache arrivals + readiness, remove, rows, cache = re-keys;
        # steps = rounds)
        for kern, opts in (("small", {}), ("warp", {"wide_min_vn": (1 << 31) - 1}), ("rounds", {"wide_min_vn": 0})):
            if kern not in kerns:
                continue
            plan = bx.Plan([gg], [job], options=dict(opts, profile=1))
            plan.upload()
            ms = []
            for _ in range(3):
                plan.place()
                ms.append(plan.kernel_ms())
            pr = plan.profile(0)
            if kern == "small" and plan.job_kernel(0) != "small-frontier":
                plan.close()
                continue
            commits = max(pr["commits"], 1)
            row = {"case": name, "kernel": kern, "V": gg.V, "n": len(job.capacity), "algo": job.algo,
                   "kernel_ms": round(min(ms), 3), "us_per_commit": round(min(ms) * 1e3 / commits, 3),
                   "steps": pr["steps"], "commits": pr["commits"], "rescans": pr["rescans"],
                   "cyc_per_commit": {k: round(pr[k] / commits, 1) for k in bx.Plan.PROFILE_FIELDS[:11]},
                   "total_cyc_per_commit": round(pr["total"] / commits, 1)}
            print(json.dumps(row), flush=True)
            plan.close()


if __name__ == "__main__":
    main()
