"""Exhaustive oracle: bx_oracle_makespan (GPU simulator,
batched) vs the reference's oracle_makespan (OpenMP over assignments) on
small random DAGs, same result required."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from oracle import Ref  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402
from test_gpu_api import _tiny_dag  # noqa: E402

rng = np.random.default_rng(5)
bx.oracle_makespan(bx.MetaGraph.from_dict(_tiny_dag(rng, 4)), 2, bx.CommModel(3.0, 0.01, 1))  # warm-up
for V, p, n in ((8, 0.3, 3), (10, 0.3, 3), (11, 0.35, 3), (12, 0.4, 3)):
    g = _tiny_dag(rng, V, p)
    gg = bx.MetaGraph.from_dict(g)
    cm = (3.0, 0.01, 1)
    t0 = time.perf_counter()
    got = bx.oracle_makespan(gg, n, bx.CommModel(*cm))
    gpu_ms = (time.perf_counter() - t0) * 1e3
    rg = Ref.graph(W.as_ref_base(g), pipeline=-1)
    t0 = time.perf_counter()
    ref = Ref.oracle_makespan(rg, n, cm)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"V": V, "E": int(g["E"]), "n": n, "gpu_ms": round(gpu_ms, 2), "cpu_ref_ms": round(cpu_ms, 2),
                      "cpu_threads": os.cpu_count(), "makespan": got, "identical": got == ref}), flush=True)
