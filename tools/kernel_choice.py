"""Per-graph kernel choice experiment: the same single-graph placement
through each eligible kernel (plan options force the dispatch; results are
identical by construction, checked here too)."""
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
    cmt = COMM_SEQ if name.startswith("seq_") else W.COMM_TEST
    cm = bx.CommModel(*cmt)
    caps = np.full(n, W.bench_capacity(g, n, f), np.int64)
    fav = fav_first(g["esrc"], g["edst"], g["V"]) if algo == "m-sct" else None
    ref = None
    for kname, opts in (("default", None), ("warp", {"wide_min_vn": (1 << 31) - 1, "no_small_frontier": 1}),
                        ("cta", {"wide_min_vn": 0, "no_small_frontier": 1})):
        plan = bx.Plan([gg], [bx.Job(0, algo, caps, cm, fav)], options=opts)
        plan.upload()
        ms = []
        for _ in range(2):
            plan.place()
            ms.append(plan.kernel_ms())
        plan.download()
        p = plan.result(0)
        same = ref is None or (np.array_equal(p.device_of, ref.device_of) and np.array_equal(p.start_us, ref.start_us))
        ref = ref or p
        print(json.dumps({"case": name, "kernel": kname, "job_kernel": plan.job_kernel(0), "ms": round(min(ms), 2),
                          "same": bool(same)}), flush=True)
        plan.close()
