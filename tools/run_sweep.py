"""Place the C5 sweep once (for ncu captures of the batch kernels)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import sweep  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

graphs, jobs = sweep.global_sweep(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
mgs = [bx.MetaGraph.from_dict(W.as_meta_dict(g)) for g in graphs]
cm = bx.CommModel(*W.COMM_TEST)
plan = bx.Plan(mgs, [bx.Job(gi, "m-etf", np.full(n, cap, np.int64), cm) for gi, n, cap in jobs])
plan.upload()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    plan.place()
    print("kernel ms", plan.kernel_ms(), flush=True)
plan.download()
