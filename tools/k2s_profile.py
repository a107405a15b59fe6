"""K2s clock64 phase breakdown per commit for latency-table cases
(python tools/k2s_profile.py refchain100k_x4 ...)."""
import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402
from latency_table import CASES, COMM_SEQ, fav_first  # noqa: E402

for name in sys.argv[1:]:
    mk, n, algo, f = CASES[name]
    g = mk()
    gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
    cm = bx.CommModel(*(COMM_SEQ if name.startswith("seq_") else W.COMM_TEST))
    caps = np.full(n, W.bench_capacity(g, n, f), np.int64)
    fav = fav_first(g["esrc"], g["edst"], g["V"]) if algo == "m-sct" else None
    plan = bx.Plan([gg], [bx.Job(0, algo, caps, cm, fav)], options={"profile": 1})
    plan.upload()
    for _ in range(2):
        plan.place()
    ms = plan.kernel_ms()
    pr = plan.profile(0)
    c = max(pr["commits"], 1)
    print(json.dumps({"case": name, "kernel": plan.job_kernel(0), "ms": round(ms, 2), "commits": pr["commits"],
                      "rounds": pr["steps"], "cyc_per_commit": {k: round(pr[k] / c) for k in bx.Plan.PROFILE_FIELDS[:11]
                                                                if pr[k]}}), flush=True)
    plan.close()
