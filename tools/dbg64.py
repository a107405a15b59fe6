import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2301_08695_b200 as bx
from paper_2301_08695_b200 import workloads as W
V = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = W.layered_dag_fast(V // 100, 100, 3)
gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
caps = np.full(n, W.bench_capacity(g, n, 1.2), np.int64)
plan = bx.Plan([gg], [bx.Job(0, "m-etf", caps, bx.CommModel(*W.COMM_TEST))])
plan.upload(); plan.place(); plan.download()
print("ok", plan.status(0), plan.kernel_ms())
