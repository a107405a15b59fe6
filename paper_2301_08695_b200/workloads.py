"""Synthetic placement workloads, generated deterministically
with numpy so the GPU path and the CPU reference consume byte-identical
graphs.

Value distributions follow the reference GenSpec defaults
(proj/include/dagsched/generator.hpp:25-34): compute U[50,150] us, tensor
U[1 KiB, 64 KiB] (same bytes on every out-edge of a node), temp U[0, 64 KiB],
perm U[1 KiB, 1 MiB], out U[1 KiB, 256 KiB]. The reference's own generator
(proj/src/generator.cpp) is O(V^2) for random DAGs and has no model-shaped
families, so these families are new; graphs are base graphs whose node ids are
0..V-1 and whose edges are sorted by (src, dst) and unique, i.e. exactly the
singleton-group meta graph (transforms.cpp:300-327) of themselves.

The comm model of the configs is proj/comm_model_test.json:1-5
(12.5 us + 0.002 us/B, parallel).
"""
from __future__ import annotations

import math

import numpy as np

COMM_TEST = (12.5, 0.002, 1)  # intercept_us, us_per_byte, mode (parallel)
KIB = 1024


def _values(rng, V):
    k = rng.integers(50, 151, V, dtype=np.int64)
    tensor = rng.integers(KIB, 64 * KIB + 1, V, dtype=np.int64)
    temp = rng.integers(0, 64 * KIB + 1, V, dtype=np.int64)
    perm = rng.integers(KIB, 1024 * KIB + 1, V, dtype=np.int64)
    out = rng.integers(KIB, 256 * KIB + 1, V, dtype=np.int64)
    return k, tensor, temp, perm, out


def _finish(V, src, dst, rng, name):
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = np.unique(src * V + dst)  # sorted by (src, dst), unique
    src, dst = key // V, key % V
    assert np.all(src < dst), "generators emit forward edges only"
    k, tensor, temp, perm, out = _values(rng, V)
    return {
        "name": name,
        "V": V,
        "k": k, "temp": temp, "perm": perm, "out": out,
        "esrc": src.astype(np.int32), "edst": dst.astype(np.int32),
        "ebytes": tensor[src],
    }


def layered_dag(layers: int, width: int, seed: int, max_parents: int = 4, reach: int = 3):
    """C4 family: `layers` x `width` nodes; each node of layer l >= 1 draws
    U{1..max_parents} distinct parents uniformly from layers [l-reach, l-1]."""
    rng = np.random.default_rng(seed)
    V = layers * width
    src, dst = [], []
    for l in range(1, layers):
        lo = max(0, l - reach) * width
        hi = l * width
        cnt = rng.integers(1, max_parents + 1, width)
        for w in range(width):
            par = rng.choice(hi - lo, size=min(int(cnt[w]), hi - lo), replace=False) + lo
            src.append(par)
            dst.append(np.full(len(par), l * width + w))
    if src:
        src, dst = np.concatenate(src), np.concatenate(dst)
    return _finish(V, src, dst, rng, f"layered{layers}x{width}")


def layered_dag_fast(layers: int, width: int, seed: int, max_parents: int = 4, reach: int = 3):
    """Vectorised layered_dag for large V (parents drawn with replacement,
    duplicates merged): the 1M-op C4 stress graph."""
    rng = np.random.default_rng(seed)
    V = layers * width
    node = np.arange(width, V, dtype=np.int64)
    layer = node // width
    cnt = rng.integers(1, max_parents + 1, len(node))
    rep = np.repeat(node, cnt)
    rl = np.repeat(layer, cnt)
    lo = np.maximum(0, rl - reach) * width
    span = rl * width - lo
    par = lo + (rng.random(len(rep)) * span).astype(np.int64)
    return _finish(V, par, rep, rng, f"layered{layers}x{width}")


def grid_chain(layers: int, width: int, seed: int, cross: float = 0.3):
    """Reference layered-chain-like family: `width` parallel chains of
    `layers` ops with random cross links to the next layer."""
    rng = np.random.default_rng(seed)
    V = layers * width
    node = np.arange(V - width, dtype=np.int64)
    src = [node, node]
    nxt = node + width
    sh = (node % width + 1) % width + (node // width + 1) * width
    mask = rng.random(len(node)) < cross
    dst = [nxt, np.where(mask, sh, nxt)]
    return _finish(V, np.concatenate(src), np.concatenate(dst), rng, f"grid{layers}x{width}")


def branchy(modules: int, seed: int, branches=(4, 6), depth=(1, 5), stem: int = 6):
    """Inception-style family (branchy, generator.cpp:59-87 shape): a stem
    chain, then `modules` split -> parallel branches -> concat modules."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    nid = 0

    def new():
        nonlocal nid
        nid += 1
        return nid - 1

    prev = new()
    for _ in range(stem - 1):
        cur = new()
        src.append(prev)
        dst.append(cur)
        prev = cur
    for _ in range(modules):
        split = new()
        src.append(prev)
        dst.append(split)
        tails = []
        for _b in range(int(rng.integers(branches[0], branches[1] + 1))):
            last = split
            for _d in range(int(rng.integers(depth[0], depth[1] + 1))):
                cur = new()
                src.append(last)
                dst.append(cur)
                last = cur
            tails.append(last)
        concat = new()
        for t in tails:
            src.append(t)
            dst.append(concat)
        prev = concat
    return _finish(nid, src, dst, rng, f"branchy{modules}")


def wide_random(V: int, seed: int, window: int = 200, fanin=(1, 3)):
    """Random DAG with bounded fan-in: node j draws U{fanin} parents from the
    `window` nodes before it."""
    rng = np.random.default_rng(seed)
    node = np.arange(1, V, dtype=np.int64)
    cnt = rng.integers(fanin[0], fanin[1] + 1, len(node))
    rep = np.repeat(node, cnt)
    lo = np.maximum(0, rep - window)
    par = lo + (rng.random(len(rep)) * (rep - lo)).astype(np.int64)
    return _finish(V, par, rep, rng, f"wide{V}")


def sweep_graphs(seed_base: int = 0, count: int = 64, vmin: int = 1000, vmax: int = 20000):
    """C5 graphs: 4 families x count/4 seeds, V spread over [vmin, vmax]."""
    out = []
    per = count // 4
    for s in range(per):
        frac = s / max(per - 1, 1)
        V = int(round(vmin + frac * (vmax - vmin)))
        seed = seed_base * 1000 + s
        w = 32 + (s % 4) * 16
        out.append(layered_dag_fast(max(2, V // w), w, 1 + seed))
        out.append(grid_chain(max(2, V // 16), 16, 2 + seed))
        out.append(branchy(max(1, V // 22), 3 + seed))
        out.append(wide_random(V, 4 + seed))
    return out


def need(g):
    return g["perm"] + g["out"] + g["temp"]


def bench_capacity(g, n: int, factor: float) -> int:
    """bench_capacity (proj/src/bench.cpp:77-87):
    ceil(factor * (total reserve / n + max reserve))."""
    nd = need(g)
    total = int(nd.sum())
    largest = int(nd.max()) if len(nd) else 0
    return int(math.ceil((float(total) / n + float(largest)) * factor))


def sweep_jobs(graphs, device_counts=(2, 4, 8, 16), factors=None):
    """C5 jobs: graph x device count x 16 capacity factors (1.05 + k*0.0633)."""
    if factors is None:
        factors = [1.05 + k * 0.0633 for k in range(16)]
    jobs = []
    for gi, g in enumerate(graphs):
        for n in device_counts:
            for f in factors:
                jobs.append((gi, n, bench_capacity(g, n, f)))
    return jobs


def as_ref_base(g):
    """The base-graph dict the oracle's reference loader takes (ids = index)."""
    V = g["V"]
    return dict(id=np.arange(V, dtype=np.int64), k=g["k"], temp=g["temp"], perm=g["perm"], out=g["out"],
                coloc=np.full(V, -1, np.int32), has_pair=np.zeros(V, np.uint8), pair=np.zeros(V, np.int64),
                src=g["esrc"].astype(np.int64), dst=g["edst"].astype(np.int64), bytes=g["ebytes"])


def as_meta_dict(g):
    return dict(V=g["V"], E=len(g["esrc"]), k=g["k"], temp=g["temp"], perm=g["perm"], out=g["out"],
                esrc=g["esrc"], edst=g["edst"], ebytes=g["ebytes"])
