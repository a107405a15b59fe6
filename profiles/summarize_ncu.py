"""Summarise ncu outputs committed under profiles/ (run here, no GPU needed).

usage: python profiles/summarize_ncu.py launches.csv [full.ncu-rep] > summary.txt
"""
import collections
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor",
        "sm__inst_executed.sum", "smsp__cycles_active.avg", "launch__shared_mem_per_block",
        "smsp__average_warp_latency_issue_stalled", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active",
        "smsp__warp_issue_stalled_barrier_per_warp_active", "smsp__warp_issue_stalled_short_scoreboard_per_warp_active",
        "smsp__warp_issue_stalled_membar_per_warp_active", "smsp__warp_issue_stalled_wait_per_warp_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum", "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e3:.1f} ms total "
          f"(ncu: serialised, cold cache — compare shares)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:6d} launches {v[1]/1e3:10.3f} ms {100*v[1]/tot:6.2f}%  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    print(f"\n# ncu --set full {path}")
    for row in r[2:]:
        kname = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## {kname[:100]}")
        for i, name in enumerate(h):
            if any(name.startswith(w) for w in WANT):
                print(f"{name:70s} {row[i]:>16s} {units[i]}")


if __name__ == "__main__":
    launches(sys.argv[1])
    for p in sys.argv[2:]:
        full(p)
