"""Which problems bound the C5 batch? Runs the sweep plan with options={"profile": 1}
and prints the longest jobs (SM cycles per job from clock64) by family/n."""
import collections
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import sweep  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402

graphs, jobs = sweep.global_sweep(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
mgs = [bx.MetaGraph.from_dict(W.as_meta_dict(g)) for g in graphs]
cm = bx.CommModel(*W.COMM_TEST)
plan = bx.Plan(mgs, [bx.Job(gi, "m-etf", np.full(n, cap, np.int64), cm) for gi, n, cap in jobs], options={"profile": 1})
plan.upload()
plan.place()
plan.download()
print("kernel ms", plan.kernel_ms())
rows = []
for i, (gi, n, cap) in enumerate(jobs):
    pr = plan.profile(i)
    rows.append((pr["total"], graphs[gi]["name"], graphs[gi]["V"], n, pr["commits"], pr["steps"]))
rows.sort(reverse=True)
clk = 1.965e9
for r in rows[:15]:
    print(f"{r[0]/clk*1e3:8.1f} ms  {r[1]:>16s} V={r[2]:6d} n={r[3]:3d} commits={r[4]} steps/rounds={r[5]}"
          f"  us/commit={r[0]/clk*1e6/max(r[4],1):.2f}")
# phase breakdown (SM cycles per commit) summed over all jobs, and over the 64 longest
tot = collections.Counter()
top = collections.Counter()
order = sorted(range(len(jobs)), key=lambda i: -plan.profile(i)["total"])
for rank, i in enumerate(order):
    pr = plan.profile(i)
    for k in bx.Plan.PROFILE_FIELDS[:11]:
        tot[k] += pr[k]
        if rank < 64:
            top[k] += pr[k]
    tot["commits"] += pr["commits"]
    if rank < 64:
        top["commits"] += pr["commits"]
for name, c in (("all jobs", tot), ("64 longest", top)):
    print(name, {k: round(c[k] / max(c["commits"], 1)) for k in bx.Plan.PROFILE_FIELDS[:11] if c[k]})
fam = collections.defaultdict(list)
for r in rows:
    fam[(r[1].rstrip('0123456789x'), r[3])].append(r[0] / clk * 1e3)
for k in sorted(fam):
    v = fam[k]
    print(k, f"max {max(v):.1f} ms mean {np.mean(v):.1f} ms")
