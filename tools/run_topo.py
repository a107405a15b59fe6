"""One m-TOPO placement of C1 (for ncu captures of k_place_topo_cta / k_acyclic)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402
gen, n, algos, kw, f = W.CONFIGS["C1_inception_mtopo_metf"]
meta, _ = bx.build_grouped(gen(), **kw)
cap = W.meta_capacity(meta, n, f)
plan = bx.Plan([meta], [bx.Job(0, "m-topo", np.full(n, cap, np.int64), bx.CommModel(*W.COMM_TEST))])
plan.upload()
for _ in range(3):
    plan.place()
    print("kernel_ms", plan.kernel_ms())
plan.close()
