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


# ---- model-shaped training graphs (configs C1-C3) ---------------------------
class _TrainGraph:
    """Builds a training DAG from forward layers: every
    forward op f gets a gradient op g_f (reversed data edges plus the
    activation edge f -> g_f, coplace_pair(f, g_f)); every layer has a weight
    Variable colocated with its reader, and a weight-gradient op colocated
    with its ApplyGrad (paper Fig. 3 colocation groups)."""

    def __init__(self, seed):
        self.rng = np.random.default_rng(seed)
        self.k, self.temp, self.perm, self.out = [], [], [], []
        self.coloc, self.pair = [], []
        self.edges = []  # (src, dst, bytes)
        self.fwd = []  # forward op ids in creation (topological) order
        self.fwd_succ = {}  # forward op -> forward consumers
        self.label = 0

    def op(self, k=None, perm=0, coloc=-1, out=None, temp=None):
        r = self.rng
        self.k.append(int(r.integers(50, 151)) if k is None else k)
        self.temp.append(int(r.integers(0, 64 * KIB + 1)) if temp is None else temp)
        self.perm.append(perm)
        self.out.append(int(r.integers(KIB, 256 * KIB + 1)) if out is None else out)
        self.coloc.append(coloc)
        self.pair.append(-1)
        return len(self.k) - 1

    def edge(self, s, d, nbytes=None):
        self.edges.append((s, d, int(self.rng.integers(KIB, 64 * KIB + 1)) if nbytes is None else nbytes))

    def fwd_op(self, inputs, weight=None):
        f = self.op()
        for i in inputs:
            self.edge(i, f)
            self.fwd_succ.setdefault(i, []).append(f)
        if weight is not None:
            self.edge(weight, f)
        self.fwd.append(f)
        self.fwd_succ.setdefault(f, [])
        return f

    def layer(self, inputs, sub):
        """`sub` forward ops in a chain; the first reads a weight Variable and
        shares its colocation_group (a Variable grouped with its ApplyGrad
        would close a cycle through the whole pass, which the reference
        rejects, transforms.cpp:343-349)."""
        lab = self.label
        self.label += 2
        v = self.op(k=1, perm=int(self.rng.integers(64 * KIB, 4096 * KIB)), coloc=lab, out=0)
        cur = self.fwd_op(inputs, weight=v)
        self.coloc[cur] = lab
        first = cur
        for _ in range(sub - 1):
            cur = self.fwd_op([cur])
        self._weights = getattr(self, "_weights", []) + [(first, v, lab)]
        return cur

    def finish(self, name):
        grad = {}
        for f in reversed(self.fwd):
            g = self.op()
            grad[f] = g
            self.edge(f, g)  # activation edge
            for c in self.fwd_succ[f]:
                self.edge(grad[c], g)  # gradient flows backwards
            self.pair[f], self.pair[g] = g, f
        for first, v, lab in getattr(self, "_weights", []):
            wg = self.op(coloc=lab + 1)  # weight gradient + ApplyGrad colocated
            self.edge(grad[first], wg)
            ap = self.op(k=20, coloc=lab + 1, out=0)
            self.edge(wg, ap)
            self.edge(v, ap, 0)
        V = len(self.k)
        es = sorted(set((s, d) for s, d, _ in self.edges))
        by = {}
        for s, d, b in self.edges:
            by.setdefault((s, d), b)
        has_pair = np.array([p >= 0 for p in self.pair], np.uint8)
        return {"name": name, "V": V, "id": np.arange(V, dtype=np.int64),
                "k": np.array(self.k, np.int64), "temp": np.array(self.temp, np.int64),
                "perm": np.array(self.perm, np.int64), "out": np.array(self.out, np.int64),
                "coloc": np.array(self.coloc, np.int32), "has_pair": has_pair,
                "pair": np.array([max(p, 0) for p in self.pair], np.int64),
                "src": np.array([s for s, _ in es], np.int64), "dst": np.array([d for _, d in es], np.int64),
                "bytes": np.array([by[e] for e in es], np.int64)}


def inception_v3(seed: int = 1, sub: int = 28):
    """C1: Inception-V3-shaped training DAG, ~7k ops: stem, 11 split ->
    branches (4-6, depth 1-5) -> concat modules, head (branchy shape,
    generator.cpp:59-87), with backward mirror, coplace pairs and
    Variable/ApplyGrad colocation."""
    t = _TrainGraph(seed)
    x = t.fwd_op([])
    for _ in range(5):
        x = t.layer([x], sub)
    for _m in range(11):
        tails = []
        for _b in range(int(t.rng.integers(4, 7))):
            y = x
            for _d in range(int(t.rng.integers(1, 4))):
                y = t.layer([y], sub)
            tails.append(y)
        x = t.fwd_op(tails)  # concat
    for _ in range(2):
        x = t.layer([x], sub)
    t.fwd_op([x])  # loss
    return t.finish(f"inception_v3_s{seed}")


def gnmt(seed: int = 1, layers: int = 4, steps: int = 40, cell_ops: int = 24):
    """C2: GNMT-shaped 4-layer LSTM seq2seq training graph, ~18k ops at
    sequence length 40: unrolled encoder/decoder cells (each a short op
    chain reading the previous step and the layer below), Bahdanau-style
    attention from every decoder step to the top encoder states, residual
    links from layer 3 up; backward mirror with coplace pairs."""
    t = _TrainGraph(seed)
    enc = [[None] * steps for _ in range(layers)]
    emb = [t.fwd_op([]) for _ in range(steps)]
    for l in range(layers):
        for s in range(steps):
            ins = [emb[s] if l == 0 else enc[l - 1][s]]
            if s > 0:
                ins.append(enc[l][s - 1])
            if l >= 2:
                ins.append(enc[l - 2][s])
            enc[l][s] = t.layer(ins, cell_ops)
    dec_prev = [None] * layers
    for s in range(steps):
        x = t.fwd_op([])  # target embedding
        att = t.fwd_op([enc[layers - 1][i] for i in range(0, steps, max(1, steps // 8))])
        for l in range(layers):
            ins = [x, att] if l == 0 else [x]
            if dec_prev[l] is not None:
                ins.append(dec_prev[l])
            x = t.layer(ins, cell_ops)
            dec_prev[l] = x
        t.fwd_op([x])  # per-step softmax / loss
    return t.finish(f"gnmt{layers}x{steps}_s{seed}")


def transformer(seed: int = 1, enc_layers: int = 6, dec_layers: int = 6, sub: int = 8):
    """C3: Transformer 6+6 module-level training graph (~2-3k ops):
    attention (q/k/v projections, scores, softmax, context, output),
    add&norm and feed-forward blocks, split into sub-ops."""
    t = _TrainGraph(seed)
    x = t.layer([t.fwd_op([])], sub)

    def attn(q_in, kv_in):
        q = t.layer([q_in], sub)
        k = t.layer([kv_in], sub)
        v = t.layer([kv_in], sub)
        sc = t.fwd_op([q, k])
        sm = t.fwd_op([sc])
        ctx = t.fwd_op([sm, v])
        o = t.layer([ctx], sub)
        return t.fwd_op([o, q_in])  # residual add + norm

    def ffn(x_in):
        h = t.layer([x_in], sub)
        y = t.layer([h], sub)
        return t.fwd_op([y, x_in])

    for _ in range(enc_layers):
        x = ffn(attn(x, x))
    memory = x
    y = t.layer([t.fwd_op([])], sub)
    for _ in range(dec_layers):
        y = attn(y, y)
        y = attn(y, memory)
        y = ffn(y)
    t.fwd_op([t.layer([y], sub)])
    return t.finish(f"transformer{enc_layers}+{dec_layers}_s{seed}")


# BASELINE.json configs[0..2] as (generator, devices, algo, pipeline, cap factor)
CONFIGS = {
    "C1_inception_mtopo_metf": (inception_v3, 4, ("m-topo", "m-etf"), dict(coplacement=True, fusion=True), 1.3),
    "C1_inception_nocoplace": (inception_v3, 4, ("m-etf",), dict(coplacement=False, fusion=False), 1.3),
    "C2_gnmt_metf_coplace": (gnmt, 4, ("m-etf",), dict(coplacement=True, fusion=True), 1.3),
    "C3_transformer_msct_tight": (transformer, 8, ("m-sct",), dict(coplacement=True, fusion=True), 1.05),
}


def meta_capacity(meta, n: int, factor: float) -> int:
    """bench_capacity (bench.cpp:77-87) on a grouped (meta) graph."""
    nd = meta.perm + meta.out + meta.temp
    return int(math.ceil((float(nd.sum()) / n + float(nd.max() if len(nd) else 0)) * factor))


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
