"""Where the one-shot drop-in call (bx_place: plan create + upload + place +
download + destroy) spends its time, on the BASELINE model configs:
median wall time of bx_place next to the same phases through a reused plan.

python tools/oneshot_profile.py [case ...]
"""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import numpy as np  # noqa: E402

import paper_2301_08695_b200 as bx  # noqa: E402
from paper_2301_08695_b200 import workloads as W  # noqa: E402
from latency_table import fav_first  # noqa: E402


def med(f, reps=15):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 4)


def main():
    want = set(sys.argv[1:])
    cm = bx.CommModel(*W.COMM_TEST)
    for name, (gen, n, algos, kw, f) in W.CONFIGS.items():
        if want and name not in want:
            continue
        meta, _ = bx.build_grouped(gen(), **kw)
        cap = np.full(n, W.meta_capacity(meta, n, f), np.int64)
        for algo in algos:
            fav = fav_first(meta.esrc, meta.edst, meta.V) if algo == "m-sct" else None
            bx._one(meta, algo, cap, cm, fav)  # warm
            row = {"case": name, "algo": algo, "V": meta.V, "oneshot_ms": med(lambda: bx._one(meta, algo, cap, cm, fav))}
            job = bx.Job(0, algo, cap, cm, fav)
            row["plan_create_destroy_ms"] = med(lambda: bx.Plan([meta], [job]).close())
            plan = bx.Plan([meta], [job])
            plan.upload()
            plan.place()
            plan.download()
            row["upload_ms"] = med(lambda: (plan.upload(), plan.download()))
            row["download_ms"] = med(lambda: plan.download())
            row["place_download_ms"] = med(lambda: (plan.place(), plan.download()))
            row["kernel_ms"] = round(plan.kernel_ms(), 4)
            row["launches"] = plan.launch_count()
            plan.close()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
