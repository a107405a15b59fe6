"""C5 sweep with and without the small-frontier kernel in the batch
(plan option no_small_frontier), kernel time per step and parity."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import sweep  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

graphs, jobs = sweep.global_sweep(64)
mgs = [bx.MetaGraph.from_dict(W.as_meta_dict(g)) for g in graphs]
cm = bx.CommModel(*W.COMM_TEST)
res = {}
for name, opts in (("k2s", None), ("no_k2s", {"no_small_frontier": 1})):
    plan = bx.Plan(mgs, [bx.Job(gi, "m-etf", np.full(n, cap, np.int64), cm) for gi, n, cap in jobs], options=opts)
    plan.upload()
    for _ in range(2):
        plan.place()
    ms = []
    for _ in range(3):
        plan.place()
        ms.append(plan.kernel_ms())
    plan.download()
    kinds = {}
    for i in range(len(jobs)):
        k = plan.job_kernel(i)
        kinds[k] = kinds.get(k, 0) + 1
    res[name] = [plan.result(i) for i in range(0, len(jobs), 7)]
    print(name, "kernel ms", [round(x, 1) for x in ms], kinds, flush=True)
    plan.close()
same = all(np.array_equal(a.device_of, b.device_of) and np.array_equal(a.start_us, b.start_us)
           for a, b in zip(res["k2s"], res["no_k2s"]))
print("same placements:", same)
