"""Run one placement case once (for ncu captures): python tools/run_case.py CASE [reps]
CASE is a CONFIGS name or grid100k_x8 / layered100k_x4 / wide100k_x16.
RC_KERNEL=small|rounds|warp selects the kernel (default: the plan's own dispatch)."""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import config_profile as CP  # noqa: E402
import paper_2301_08695_b200 as bx  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for nm, gg, job in CP.cases():
    if nm != name:
        continue
    kern = os.environ.get("RC_KERNEL", "")
    opts = {"small": None, "rounds": {"wide_min_vn": 0}, "warp": {"wide_min_vn": (1 << 31) - 1}}.get(kern)
    plan = bx.Plan([gg], [job], options=opts)
    plan.upload()
    for _ in range(reps):
        plan.place()
        print(name, "kernel_ms", plan.kernel_ms(), flush=True)
    plan.close()
    break
