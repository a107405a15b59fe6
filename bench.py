"""Benchmark: batched m-ETF placements/sec on the C5 sweep (BASELINE.json
configs[4]), plus the reference CPU placer timed on this box's host cores.

python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]

One process per GPU (torchrun for N > 1). Every rank holds the SAME global
sweep (64 graphs x {2,4,8,16} devices x 16 memory caps = 4096 problems) and
places its longest-processing-time share (cost V*n), so the
total work is fixed as N grows ("strong"). A "step" is one pass of the
placement engine over the whole sweep; the job time is the slowest rank's.
`value` is device-resident (inputs already in HBM); `e2e` re-uploads every
input from pinned host memory, places, and brings every placement to the
host through the C ABI (bx_plan_upload / bx_plan_place / bx_plan_download),
with the NCCL gather of all ranks' placements to rank 0 inside the step for
N > 1. After timing, rank 0 compares all 4096 placements (device_of,
start_us, exec_order, exec_off, stats, status) with the reference's.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "batched placements/sec"
UNIT = "placements/s"
PEAKS = os.path.join(HERE, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(HERE, "profiles", "ncu_placer_summary.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes(graphs, jobs):
    """B = 40 V + 16 E per placement (m-ETF)."""
    return sum(40 * graphs[g]["V"] + 16 * len(graphs[g]["esrc"]) for g, _, _ in jobs)


def stratified(P, stride, offset=0):
    """Every stride-th problem with a rotating offset: jobs are ordered
    (graph, devices, cap) with the 16 caps innermost, so a plain stride would
    always pick the same cap factor; this one cycles through all of them."""
    return [i for i in range(P) if i % stride == (i // stride + offset) % stride]


def cpu_reference(graphs, jobs, idx, threads, full=False):
    """The reference placer (oracle/_ref = the unmodified reference sources)
    over problems `idx` with the reference's own sweep pattern, OpenMP over
    problems (proj/src/bench.cpp:121). Returns (placements/s, statuses,
    placements or None)."""
    from oracle import Ref
    from paper_2301_08695_b200 import workloads as W
    if not Ref.available():
        raise RuntimeError("oracle/_ref/libdagsched_ref.so missing (build with make -C oracle)")
    used = sorted({jobs[i][0] for i in idx})
    rg = {g: Ref.graph(W.as_ref_base(graphs[g]), -1) for g in used}
    maxn = max(jobs[i][1] for i in idx)
    caps = np.zeros((len(idx), maxn), np.int64)
    for r, i in enumerate(idx):
        caps[r, :jobs[i][1]] = jobs[i][2]
    gl = [rg[jobs[i][0]] for i in idx]
    algos = np.ones(len(idx), np.int32)
    ns = np.array([jobs[i][1] for i in idx], np.int32)
    if full:
        st, pls, wall_ns = Ref.place_batch_full(gl, algos, ns, caps, W.COMM_TEST, threads)
    else:
        st, _, wall_ns = Ref.place_batch(gl, algos, ns, caps, W.COMM_TEST, threads)
        pls = None
    return len(idx) / (wall_ns / 1e9), st, pls


def compare_all(results, ref_status, ref_pls, idx):
    """Full-placement parity of every problem in idx against the reference."""
    mism = []
    for r, i in enumerate(idx):
        got = results[i]
        if int(ref_status[r]) != got["status"]:
            mism.append(i)
            continue
        if ref_status[r] != 0:
            continue
        o = ref_pls[r]
        if not (np.array_equal(o.device_of, got["device_of"]) and np.array_equal(o.start_us, got["start_us"])
                and np.array_equal(o.exec_order, got["exec_order"]) and np.array_equal(o.exec_off, got["exec_off"])
                and np.array_equal(np.asarray(o.stats), got["stats"])):
            mism.append(i)
    return mism


def per_graph(bx, W, cpu=True):
    """Placement wall time per graph (the metric's first half): a 100k-op
    random layered DAG (C4 family, 100 layers x 1000), 4 devices, m-ETF,
    comm_model_test.json. GPU = placer kernel on device-resident inputs
    (CUDA events, best of 3 after a warm-up) and end to end through the C ABI
    (upload + place + download); CPU = the compiled reference place_metf on
    one host core (run_placer's scope), same graph, bit-exact compared."""
    import time as _t
    g = W.layered_dag_fast(100, 1000, 3)
    gg = bx.MetaGraph.from_dict(W.as_meta_dict(g))
    cm = bx.CommModel(*W.COMM_TEST)
    caps = np.full(4, W.bench_capacity(g, 4, 1.2), np.int64)
    plan = bx.Plan([gg], [bx.Job(0, "m-etf", caps, cm)])
    plan.upload()
    ks = []
    for _ in range(4):
        plan.place()
        ks.append(plan.kernel_ms())
    e2e = []
    for _ in range(2):
        t0 = _t.perf_counter()
        plan.upload()
        plan.place()
        plan.download()
        e2e.append((_t.perf_counter() - t0) * 1e3)
    p = plan.result(0)
    # the makespan simulator (K4f) scoring this placement, device-resident
    import torch
    sims = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        plan.simulate(1)
        torch.cuda.synchronize()
        sims.append((_t.perf_counter() - t0) * 1e3)
    rep = plan.sim_download()[0]
    out = {"workload": "layered DAG 100 x 1000 (V=100k, E=%d), 4 devices, m-etf, parallel comm" % gg.E,
           "gpu_kernel_ms": min(ks[1:]), "gpu_e2e_ms": min(e2e), "gpu_sim_ms": min(sims[1:])}
    plan.close()
    if cpu:
        from oracle import Ref
        rg = Ref.graph(W.as_ref_base(g), -1)
        o = Ref.place(rg, 1, caps, W.COMM_TEST)
        out["cpu_ref_ms"] = o.wall_ns / 1e6
        out["cpu_cores"] = 1
        out["bit_exact"] = bool(np.array_equal(o.device_of, p.device_of) and np.array_equal(o.start_us, p.start_us)
                                and np.array_equal(o.exec_order, p.exec_order_flat))
        out["speedup_kernel"] = out["cpu_ref_ms"] / out["gpu_kernel_ms"]
        out["speedup_e2e"] = out["cpu_ref_ms"] / out["gpu_e2e_ms"]
        so = Ref.simulate(rg, caps, W.COMM_TEST, 1, o.device_of, o.exec_order, o.exec_off)
        out["cpu_ref_sim_ms"] = so.wall_ns / 1e6
        out["sim_bit_exact"] = bool(so.makespan == rep.makespan_us and np.array_equal(so.start_us, rep.start_us)
                                    and so.peak.tolist() == rep.peak_bytes.tolist())
        out["speedup_sim"] = out["cpu_ref_sim_ms"] / out["gpu_sim_ms"]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--graphs", type=int, default=64)
    ap.add_argument("--ref-stride", type=int, default=8, help="reference arm: every k-th problem per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-per-graph", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2301_08695_b200 import sweep
    from paper_2301_08695_b200 import workloads as W

    graphs, jobs = sweep.global_sweep(args.graphs)
    P = len(jobs)
    config = {"workload": "C5 batched sweep: 64 graphs (layered/grid/branchy/wide, V 1k-20k) x "
                          "{2,4,8,16} devices x 16 caps (1.05+k*0.0633), m-ETF, comm_model_test.json "
                          "(12.5us + 0.002us/B, parallel)",
              "problems": P, "partition": "LPT by V*n over ranks (same problems at every N)", "algo": "m-etf",
              "l2": "inputs+workspace larger than L2 (GBs, rewritten every step)"}

    if args.impl == "reference":
        # the reference's own sweep (oracle/_ref, unmodified sources): OpenMP
        # over problems on every host thread, one stratified sample per step
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        stride = max(1, args.ref_stride)
        for w in range(args.warmup):
            cpu_reference(graphs, jobs, stratified(P, stride * 4, w), threads)
        rates = [cpu_reference(graphs, jobs, stratified(P, stride, k), threads)[0] for k in range(args.steps)]
        v = statistics.median(rates)
        n_step = len(stratified(P, stride, 0))
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": P / v * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
                "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                 "cpu_model": cpu_model(),
                                 "sample": f"{n_step} of the {P} sweep problems per step (every {stride}th, "
                                           f"offset rotating through the cap factors), reference place_metf, "
                                           f"OpenMP over problems"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2301_08695_b200 as bx
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    ids, sgraphs, sjobs = sweep.rank_shard(rank, world, graphs, jobs)
    PR = len(ids)
    keep = []

    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        keep.append(t)
        return t.numpy()

    mgs = []
    for g in sgraphs:
        mgs.append(bx.MetaGraph(pinned(g["k"]), pinned(g["temp"]), pinned(g["perm"]), pinned(g["out"]),
                                pinned(g["esrc"]), pinned(g["edst"]), pinned(g["ebytes"])))
    for m in mgs:  # adjacency arrays pinned too
        m.in_off, m.in_edge, m.out_off = pinned(m.in_off), pinned(m.in_edge), pinned(m.out_off)
    cm = bx.CommModel(*W.COMM_TEST)
    bjobs = [bx.Job(gi, "m-etf", pinned(np.full(n, cap, np.int64)), cm) for gi, n, cap in sjobs]
    t0 = time.time()
    plan = bx.Plan(mgs, bjobs, device=local)
    log(f"[rank {rank}] plan: {PR} of {P} problems (LPT cost {sum(sgraphs[g]['V'] * n for g, n, _ in sjobs)}), "
        f"{sum(g['V'] for g in sgraphs)} graph nodes, created in {time.time() - t0:.2f}s")
    h2d = sum(m.k.nbytes + m.temp.nbytes + m.perm.nbytes + m.out.nbytes + m.esrc.nbytes + m.edst.nbytes
              + m.ebytes.nbytes + m.in_off.nbytes + m.in_edge.nbytes + m.out_off.nbytes for m in mgs)
    h2d += sum(8 * n for _, n, _ in sjobs)
    d2h = plan.output_region()[1]
    table = sweep.offsets_table(plan, ids)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return sweep.max_over_ranks(x, dist, dev)

    def gather():
        """Every rank's device-resident placements to rank 0 over NCCL."""
        return sweep.gather_to_root(sweep.region_tensor(plan, dev), table, dist, dev)

    plan.upload(sp)
    for _ in range(args.warmup):
        plan.upload(sp)
        plan.place(sp)
        plan.download(sp)
    fails = [i for i in range(PR) if plan.status(i)[0] not in (0, 3)]
    if fails:
        raise RuntimeError(f"problems failed: {[plan.status(i) for i in fails[:3]]}")

    # ---- device-resident timed region -----------------------------------
    # serial: one plan, steps back to back (the placer-kernel events of these
    # steps give the roofline's kernel time)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        plan.place(sp)
    ev1.record(stream)
    ev1.synchronize()
    serial_ms = max_over_ranks(ev0.elapsed_time(ev1))
    kernel_ms = plan.kernel_times(args.steps)
    # pipelined: two plans on two streams (every rank), steps alternating, so
    # one step's last long problems share the GPU with the next step's first
    # ones; the clock runs from the first launch to the later of the two
    # streams' last
    plan2 = bx.Plan(mgs, bjobs, device=local)
    st2 = torch.cuda.Stream()
    sp2 = st2.cuda_stream
    plan2.upload(sp2)
    for _ in range(max(args.warmup, 1)):
        plan2.place(sp2)
    plan2.download(sp2)
    lanes = [(plan, sp), (plan2, sp2)]
    barrier()
    with Clocks(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev2 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        st2.wait_event(ev0)
        for i in range(args.steps):
            lanes[i % 2][0].place(lanes[i % 2][1])
        ev1.record(stream)
        ev2.record(st2)
        torch.cuda.synchronize()
        dev_ms = max(ev0.elapsed_time(ev1), ev0.elapsed_time(ev2))
    barrier()
    rank_ms = dev_ms / args.steps
    busy = [rank_ms]
    if dist is not None:
        t = torch.tensor([rank_ms], dtype=torch.float64, device=dev)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        busy = [float(x.item()) for x in parts]
    ms_step = max(busy)
    launches = plan.launch_count() * args.steps
    value = P / (ms_step / 1e3)

    # ---- end to end through the C ABI with host buffers --------------------
    # one process per GPU: the same two plans, so step i+1's upload and
    # placement overlap step i's download (every step still moves its inputs
    # host->device and its whole output region device->host, pinned)
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        if dist is not None:
            plan.upload(sp)
            plan.place(sp)
            got = gather()
            if rank == 0:
                plan.download(sp)
        else:
            p_, s_ = lanes[i % 2]
            p_.upload(s_)  # waits for this plan's previous step (the other one keeps the GPU busy)
            p_.place(s_)
            p_.download_async(s_)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    barrier()
    e2e_ms = max_over_ranks(e2e_ms)
    e2e_value = P / (e2e_ms / args.steps / 1e3)

    # ---- the final gather on its own (full placements to rank 0) ----------
    barrier()
    gather_ms = None
    g0 = time.perf_counter()
    if dist is not None:
        gathered = gather()
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - g0) * 1e3
    else:
        torch.cuda.synchronize()
        region = sweep.region_tensor(plan, dev).cpu().numpy()
        gathered = [(region, table)]
    results = None
    if rank == 0:
        sizes = lambda i: (graphs[jobs[i][0]]["V"], jobs[i][1])  # noqa: E731
        results = sweep.collect(gathered, sizes)
        assert sorted(results) == list(range(P)), "gather lost problems"
    infeasible = None if results is None else sum(1 for r in results.values() if r["status"] == 3)

    # ---- roofline of the dominant kernel (the placer) ------------------------
    kmean = statistics.mean(kernel_ms)
    abytes = algorithmic_bytes(sgraphs, sjobs)
    achieved = abytes / (kmean / 1e3) / 1e9
    peak = None
    peak_src = "fallback 6650 GB/s (B200_PROFILING.md)"
    try:
        peak = json.load(open(PEAKS))["hbm_gbs"]
        peak_src = "measured MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        peak = 6650.0
    traffic = None
    try:
        traffic = json.load(open(NCU_SUMMARY)).get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---- parity of EVERY problem vs the reference; CPU baselines ---------------
    cpu = None
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            threads = os.cpu_count() or 1
            rate, st, pls = cpu_reference(graphs, jobs, list(range(P)), threads, full=True)
            mism = compare_all(results, st, pls, list(range(P)))
            parity = {"checked": P, "fields": "status, device_of, start_us, exec_order, exec_off, stats",
                      "mismatches": len(mism), "first_mismatches": mism[:5]}
            if world == 1 and not args.no_cpu_baseline:
                one_idx = stratified(P, 64)
                rate1, _, _ = cpu_reference(graphs, jobs, one_idx, 1)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                       "cpu_model": cpu_model(),
                       "sample": f"all {P} sweep problems, reference place_metf, OpenMP over problems "
                                 f"(the run parity is checked on)",
                       "single_thread_value": rate1,
                       "single_thread_sample": f"{len(one_idx)} problems (every 64th, rotating cap factor), 1 thread"}
        except Exception as e:  # the baseline is reported, never the target
            parity = {"error": str(e)}

    pg = None
    if rank == 0 and world == 1 and not args.no_per_graph:
        try:
            pg = per_graph(bx, W, cpu=not args.no_cpu_baseline)
        except Exception as e:
            pg = {"error": str(e)}
        # BASELINE configs C1-C3 (single model-shaped graphs): GPU placer
        # kernels (device-resident) and the one-shot bx_place call, next to the
        # reference placer on one core (median of 10), bit-exact flag
        try:
            sys.path.insert(0, os.path.join(HERE, "tools"))
            from latency_table import run_config
            pg["configs"] = [
                {k: r.get(k) for k in ("case", "algo", "meta_V", "n", "kernel", "gpu_kernel_ms", "gpu_oneshot_ms",
                                       "cpu_ref_ms", "bit_exact", "speedup", "speedup_oneshot")}
                for name in W.CONFIGS for r in run_config(name, cpu=not args.no_cpu_baseline)]
        except Exception as e:
            pg["configs"] = {"error": str(e)}
        # other 100k-op families next to the reference on one core: the
        # reference's own layered-chain (4-wide frontier), 16 chains, a wide
        # random DAG, 64 devices, and sequential comm mode
        try:
            from latency_table import run as run_case
            pg["families"] = [run_case(nm, cpu=not args.no_cpu_baseline)
                              for nm in ("refchain100k_x4", "refchain100k_x8", "refchain1M_x64", "refchain100k_x4_sct",
                                         "refchain100k_x8_sct", "grid100k_x8",
                                         "wide100k_x16",
                                         "layered100k_x64",
                                         "seq_layered100k_x4", "seq_wide100k_x16", "seq_refchain100k_x4")]
        except Exception as e:
            pg["families"] = {"error": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": config,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "note": "rank 0's numbers; each rank uploads its shard, rank 0 downloads all"
                                if world > 1 else "upload + place + download per step; two plans on two streams "
                                                  "overlap step i+1's upload/placement with step i's download"},
                "gpu_launches": launches,
                "pipelining": {"steps_in_flight": 2,
                               "serial_value": P / (serial_ms / args.steps / 1e3),
                               "serial_ms_per_step": serial_ms / args.steps,
                               "note": "value: two plans on two streams, steps alternating (one step's last "
                                       "long problems share the GPU with the next step's first); serial_value: "
                                       "one plan, steps back to back"},
                "ranks": {"busy_ms_per_step": busy, "imbalance": max(busy) / (sum(busy) / len(busy)),
                          "gather_ms": gather_ms},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "kernel": "k_place_list", "kernel_ms": kmean,
                             "algorithmic_bytes_per_launch": abytes, "peak_source": peak_src,
                             "note": "latency-bound dependent scheduling chain; bytes = 40V+16E per problem"},
                "cpu_baseline": cpu, "parity_vs_reference": parity, "infeasible_problems": infeasible,
                "clocks": clk.summary(), "per_graph": pg}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    plan.close()


if __name__ == "__main__":
    main()
