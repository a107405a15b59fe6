"""m-SCT front half timing: build_lp + solve_relaxed (bx_lp_solve: host IPM,
GPU sparse Cholesky) + round_and_extract (K3) on C3 and larger DAGs, with
HiGHS (scipy) objective cross-checks where it finishes quickly."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

cm = bx.CommModel(*W.COMM_TEST)
cases = []
gen, n, algos, kw, f = W.CONFIGS["C3_transformer_msct_tight"]
meta, _ = bx.build_grouped(gen(), **kw)
cases.append(("C3_transformer", meta))
for V, w in ((2000, 40), (6000, 60)):
    g = W.layered_dag_fast(V // w, w, 5)
    cases.append((f"layered{V // 1000}k", bx.MetaGraph.from_dict(W.as_meta_dict(g))))
for name, gg in cases:
    t0 = time.perf_counter()
    fc, fp, st, sol = bx.sct_favorites(gg, cm, 0.1)
    ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"case": name, "V": gg.V, "E": gg.E, "lp_rows": sol.rows["total"], "iterations": sol.iterations,
                      "w": sol.w, "rel_gap": sol.rel_gap, "favorite_edges": int(st[0]), "repaired": int(st[1]),
                      "sct_front_ms": round(ms, 1)}), flush=True)
