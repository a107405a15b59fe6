"""Per-step latency breakdown of the list placer (clock64 instrumentation).

python tools/step_profile.py [workload]
Prints, per job, the SM cycles per committed step spent in each phase.
"""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import paper_2301_08695_b200 as bx
from paper_2301_08695_b200 import workloads as W

which = sys.argv[1] if len(sys.argv) > 1 else "sweep-big"
cm = bx.CommModel(*W.COMM_TEST)
if which == "sweep-big":
    gs = W.sweep_graphs(0, 64)[-4:]
    cases = [(g, n) for g in gs for n in (4, 16)]
elif which == "c4":
    g = W.layered_dag_fast(1000, 1000, 1)
    cases = [(g, 64)]
elif which == "n64":
    g = W.layered_dag_fast(100, 100, 3)
    cases = [(g, 16), (g, 32), (g, 64)]
elif which == "grid":
    g = W.grid_chain(6250, 16, 4)
    cases = [(g, 8)]
else:
    g = W.layered_dag_fast(100, 1000, 1)
    cases = [(g, 4), (g, 8)]
graphs = []
jobs = []
for gi, (g, n) in enumerate(cases):
    graphs.append(bx.MetaGraph.from_dict(W.as_meta_dict(g)))
    jobs.append(bx.Job(gi, "m-etf", np.full(n, W.bench_capacity(g, n, 1.3), np.int64), cm))
res = []
for gi in range(len(cases)):
    plan = bx.Plan([graphs[gi]], [bx.Job(0, "m-etf", jobs[gi].capacity, cm)], options={"profile": 1})
    plan.upload()
    plan.place()
    plan.download()
    ms = plan.kernel_ms()
    pr = plan.profile(0)
    steps = max(pr["commits"], 1)
    rounds = max(pr["steps"], 1)
    row = {"graph": cases[gi][0]["name"], "V": graphs[gi].V, "n": len(jobs[gi].capacity), "kernel_ms": ms,
           "us_per_commit": ms * 1e3 / steps, "steps_or_rounds": pr["steps"], "commits_per_round": round(steps / rounds, 2), "rescans": pr["rescans"],
           "cycles_per_commit": {k: round(pr[k] / steps, 1) for k in bx.Plan.PROFILE_FIELDS[:11]}}
    res.append(row)
    print(json.dumps(row), flush=True)
    plan.close()
