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
# warm-up: CUDA context and module load stay out of the timed cases
bx.sct_favorites(bx.MetaGraph.from_dict(W.as_meta_dict(W.branchy(2, 1))), cm)
cases = []
for cname in ("C3_transformer_msct_tight", "C1_inception_mtopo_metf", "C2_gnmt_metf_coplace"):
    gen, n, algos, kw, f = W.CONFIGS[cname]
    meta, _ = bx.build_grouped(gen(), **kw)
    cases.append((cname.split("_")[0] + "_" + cname.split("_")[1], meta))
# model-shaped graphs at 100k base ops (after co-placement + fusion)
for name, g in (("transformer_100k", W.transformer(enc_layers=300, dec_layers=300)),):
    meta, _ = bx.build_grouped(g, coplacement=True, fusion=True)
    cases.append((name, meta))
# a random layered DAG: heavy fill (no update lists; sequential factorization)
g = W.layered_dag_fast(2000 // 40, 40, 5)
cases.append(("layered2k", bx.MetaGraph.from_dict(W.as_meta_dict(g))))
for name, gg in cases:
    t0 = time.perf_counter()
    fc, fp, st, sol = bx.sct_favorites(gg, cm, 0.1)
    ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"case": name, "V": gg.V, "E": gg.E, "lp_rows": sol.rows["total"], "iterations": sol.iterations,
                      "w": sol.w, "rel_gap": sol.rel_gap, "favorite_edges": int(st[0]), "repaired": int(st[1]),
                      "sct_front_ms": round(ms, 1), "solver": sol.solver,
                      # favourite-map stability: relaxed x values near the 0.1 rounding threshold
                      "x_within_1e-3_of_thr": int(np.sum(np.abs(sol.x - 0.1) < 1e-3)),
                      "x_within_1e-6_of_thr": int(np.sum(np.abs(sol.x - 0.1) < 1e-6)),
                      "min_abs_x_minus_thr": float(np.min(np.abs(sol.x - 0.1))) if len(sol.x) else None}),
          flush=True)
