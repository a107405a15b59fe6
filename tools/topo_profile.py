import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2301_08695_b200 as bx
from paper_2301_08695_b200 import workloads as W
gen, n, algos, kw, f = W.CONFIGS["C1_inception_mtopo_metf"]
meta, _ = bx.build_grouped(gen(), **kw)
cap = W.meta_capacity(meta, n, f)
plan = bx.Plan([meta], [bx.Job(0, "m-topo", np.full(n, cap, np.int64), bx.CommModel(*W.COMM_TEST))], options={"profile": 1})
plan.upload()
for _ in range(3):
    plan.place(); print("kernel_ms", plan.kernel_ms())
pr = plan.profile(0)
print({k: round(v / 1965.0, 1) for k, v in list(pr.items())[:5]}, "us")
