"""K4 simulator timing on a 100k-op placement vs the reference simulate()."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2301_08695_b200 as bx
from paper_2301_08695_b200 import workloads as W
from oracle import Ref

g = W.layered_dag_fast(100, 1000, 3)
gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
cm = bx.CommModel(*W.COMM_TEST)
caps = np.full(4, W.bench_capacity(g, 4, 1.2), np.int64)
plan = bx.Plan([gg], [bx.Job(0, "m-etf", caps, cm)])
plan.upload(); plan.place(); plan.download()
p = plan.result(0)
for mm in (1, 0):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        plan.simulate(mm); reps = plan.sim_download()
        ts.append((time.perf_counter() - t0) * 1e3)
    r = reps[0]
    rg = Ref.graph(W.as_ref_base(g), -1)
    o = Ref.simulate(rg, caps, W.COMM_TEST, mm, p.device_of, p.exec_order_flat, p.exec_off)
    print(json.dumps({"mem_mode": mm, "gpu_sim_ms": min(ts), "cpu_ref_sim_ms": o.wall_ns / 1e6,
                      "same": bool(o.makespan == r.makespan_us and np.array_equal(o.start_us, r.start_us)
                                   and o.peak.tolist() == r.peak_bytes.tolist())}))
