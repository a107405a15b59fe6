"""K4 simulator timing on a 100k-op placement vs the reference simulate():
device time of bx_plan_simulate (CUDA events on its stream) and the wall time
including the report download."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from oracle import Ref  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
seq = len(sys.argv) > 2 and sys.argv[2] == "seq"  # sequential comm: the event-loop kernel (K4)
g = W.layered_dag_fast(100, 1000, 3)
gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
COMM = (5.0, 0.001, 0) if seq else W.COMM_TEST
cm = bx.CommModel(*COMM)
caps = np.full(n, W.bench_capacity(g, n, 1.2), np.int64)
plan = bx.Plan([gg], [bx.Job(0, "m-etf", caps, cm)])
plan.upload()
plan.place()
plan.download()
p = plan.result(0)
st = torch.cuda.current_stream()
for mm in (1, 0):
    dev, wall = [], []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(st)
        plan.simulate(mm, st.cuda_stream)
        e1.record(st)
        reps = plan.sim_download(st.cuda_stream)
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
    r = reps[0]
    rg = Ref.graph(W.as_ref_base(g), -1)
    o = Ref.simulate(rg, caps, COMM, mm, p.device_of, p.exec_order_flat, p.exec_off)
    print(json.dumps({"n": n, "comm": "sequential" if seq else "parallel", "mem_mode": mm, "gpu_sim_device_ms": min(dev[1:]), "gpu_sim_wall_ms": min(wall[1:]),
                      "cpu_ref_sim_ms": o.wall_ns / 1e6,
                      "same": bool(o.makespan == r.makespan_us and np.array_equal(o.start_us, r.start_us)
                                   and o.peak.tolist() == r.peak_bytes.tolist())}), flush=True)
