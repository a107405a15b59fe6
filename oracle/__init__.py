"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the two parity oracles.

* ``Ref``     — the unmodified reference C++ sources compiled by
  ``oracle/Makefile`` into ``oracle/_ref/libdagsched_ref.so`` (see
  ``oracle/ref_driver.cpp`` for the entry points it forwards to).
* ``Restate`` — the plain-C restatement ``oracle/restate.c`` built into
  ``oracle/_build/librestate.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package; the product (``paper_2301_08695_b200``) never
does, and never falls back to it.

Graphs cross this boundary as plain numpy arrays:

* base graph: dict with ``id, k, temp, perm, out`` (int64), ``coloc`` (int32,
  -1 = no colocation_group), ``has_pair`` (uint8), ``pair`` (int64),
  ``src, dst, bytes`` (int64 node ids / bytes);
* meta graph: dict with ``k, temp, perm, out`` (int64 [V]), ``esrc, edst``
  (int32 [E], sorted by (src, dst)), ``ebytes`` (int64 [E]) and optional
  ``first_id`` (int64 [V]).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_ERRLEN = 1 << 20  # error-text buffers: a CycleError lists every residue group id

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libdagsched_ref.so")
RESTATE_SO = os.path.join(HERE, "_build", "librestate.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class OracleError(Exception):
    def __init__(self, kind: int, msg: str):
        super().__init__(msg)
        self.kind = kind
        self.msg = msg


def build(ref: bool = True) -> None:
    """Builds the restatement (always) and the reference (when present)."""
    target = "all" if ref else "restate"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _a(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def _opt(x, dt):
    return None if x is None else _a(x, dt)


class Placement:
    def __init__(self, device_of, start_us, exec_order, exec_off, stats=None, wall_ns=None):
        self.device_of = device_of
        self.start_us = start_us
        self.exec_order = exec_order
        self.exec_off = exec_off
        self.stats = stats
        self.wall_ns = wall_ns

    def exec_lists(self):
        return [list(self.exec_order[self.exec_off[d]:self.exec_off[d + 1]])
                for d in range(len(self.exec_off) - 1)]


class SimResult:
    def __init__(self, makespan, start_us, dev3n, xfer4, wall_ns=None):
        self.makespan = int(makespan)
        self.start_us = start_us
        self.peak = dev3n[0::3].copy()
        self.busy = dev3n[1::3].copy()
        self.idle = dev3n[2::3].copy()
        self.transfer_count, self.transfer_bytes, self.duplicate_transfers, self.cache_hits = (
            int(v) for v in xfer4)
        self.wall_ns = wall_ns


# --------------------------------------------------------------------------
class Ref:
    """The reference itself (proj/src/*.cpp), compiled in place."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(REF_SO)
            cp, ip = C.c_char_p, C.c_int
            L.ref_graph_new.argtypes = [C.c_int32, _i64p, _i64p, _i64p, _i64p, _i64p, _i32p,
                                        _u8p, _i64p, C.c_int32, _i64p, _i64p, _i64p, C.c_int32,
                                        C.POINTER(C.c_void_p), cp, ip]
            L.ref_graph_free.argtypes = [C.c_void_p]
            L.ref_graph_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int32)] * 5
            L.ref_graph_meta.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p, _i32p, _i32p,
                                         _i64p, _i32p, _i32p, _i32p, _i32p]
            L.ref_graph_base.argtypes = [C.c_void_p, _i64p, _i32p, _i32p, _i64p]
            L.ref_meta_topo_order.argtypes = [C.c_void_p, _i32p, cp, ip]
            L.ref_critical_path.argtypes = [C.c_void_p]
            L.ref_critical_path.restype = C.c_int64
            L.ref_comm_time.argtypes = [C.c_double, C.c_double, C.c_int64,
                                        C.POINTER(C.c_int64), cp, ip]
            L.ref_max_comm_time.argtypes = [C.c_void_p, C.c_double, C.c_double]
            L.ref_max_comm_time.restype = C.c_int64
            L.ref_bench_capacity.argtypes = [C.c_void_p, C.c_int32, C.c_double]
            L.ref_bench_capacity.restype = C.c_int64
            L.ref_place.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _i64p, C.c_double,
                                    C.c_double, C.c_int32, C.c_void_p, _i32p, _i64p, _i32p,
                                    _i32p, _i64p, C.POINTER(C.c_int64), cp, ip]
            L.ref_place_timed.argtypes = [C.c_void_p, C.c_int32, C.c_int32, _i64p, C.c_double,
                                          C.c_double, C.c_int32, C.c_void_p, C.c_int32, _i64p,
                                          cp, ip]
            L.ref_place_batch.argtypes = [C.c_int32, C.POINTER(C.c_void_p), _i32p, _i32p, _i64p,
                                          C.c_int32, C.c_double, C.c_double, C.c_int32,
                                          C.c_int32, _i32p, _i64p, C.POINTER(C.c_int64)]
            L.ref_schedulable_time.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_double,
                                               C.c_double, _i64p, _i64p, _i32p, _i64p, _i64p,
                                               C.c_int32, C.c_int32, C.POINTER(C.c_int64), cp, ip]
            L.ref_simulate.argtypes = [C.c_void_p, C.c_int32, _i64p, C.c_double, C.c_double,
                                       C.c_int32, C.c_int32, _i32p, _i32p, _i32p,
                                       C.POINTER(C.c_int64), _i64p, _i64p, _i64p,
                                       C.POINTER(C.c_int64), cp, ip]
            L.ref_generate.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                       C.c_uint64, C.c_void_p, C.c_double, C.c_double, C.c_int32,
                                       C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, cp, ip]
            i64p, vp = C.POINTER(C.c_int64), C.c_void_p
            L.ref_simulate_trace_csv.argtypes = [vp, C.c_int32, _i64p, C.c_double, C.c_double, C.c_int32,
                                                 C.c_int32, _i32p, _i32p, _i32p, vp, C.c_int64, i64p, i64p,
                                                 cp, ip]
            L.ref_graph_json_roundtrip.argtypes = [cp, C.c_int64, vp, C.c_int64, i64p, cp, ip]
            L.ref_graph_to_json.argtypes = [vp, vp, C.c_int64, i64p]
            L.ref_comm_model_roundtrip.argtypes = [cp, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                   C.POINTER(C.c_int32), vp, C.c_int64, i64p, cp, ip]
            L.ref_placement_to_json.argtypes = [vp, cp, C.c_int32, _i32p, _i32p, _i32p, _i64p, C.c_int64, _i64p,
                                                vp, C.c_int64, i64p]
            L.ref_placement_from_json.argtypes = [vp, cp, C.c_int64, C.c_int32, cp, ip, _i32p, _i64p, _i32p,
                                                  _i32p, cp, ip]
            L.ref_place_batch_full.argtypes = [C.c_int32, C.POINTER(C.c_void_p), _i32p, _i32p, _i64p, C.c_int32,
                                               C.c_double, C.c_double, C.c_int32, C.c_int32, _i64p, _i64p, _i32p,
                                               _i64p, _i32p, _i32p, _i64p, _i32p, C.POINTER(C.c_int64)]
            L.ref_oracle_makespan.argtypes = [vp, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int64, C.c_int32,
                                              C.c_int32, C.c_int32, C.c_int64, i64p, cp, ip]
            cls._lib = L
        return cls._lib

    @classmethod
    def place_batch_full(cls, graphs, algos, ns, caps2d, cm, threads=0):
        """ref_place_batch_full: every problem's full placement. Returns
        (status [P], list of Placement | None, wall_ns)."""
        count = len(graphs)
        arr = (C.c_void_p * count)(*[g.h for g in graphs])
        Vs = np.array([g.sizes()[2] for g in graphs], np.int64)
        ns = _a(ns, np.int32)
        voff = np.zeros(count, np.int64)
        voff[1:] = np.cumsum(Vs)[:-1]
        eoff = np.zeros(count, np.int64)
        eoff[1:] = np.cumsum(ns.astype(np.int64) + 1)[:-1]
        tv = int(Vs.sum())
        dev, st, eo = np.zeros(max(tv, 1), np.int32), np.zeros(max(tv, 1), np.int64), np.zeros(max(tv, 1), np.int32)
        off = np.zeros(int((ns.astype(np.int64) + 1).sum()), np.int32)
        stats = np.zeros(3 * count, np.int64)
        status = np.zeros(count, np.int32)
        wall = C.c_int64()
        caps2d = _a(caps2d, np.int64)
        cls.lib().ref_place_batch_full(count, arr, _a(algos, np.int32), ns, caps2d, caps2d.shape[1], cm[0], cm[1],
                                       cm[2], threads, voff, eoff, dev, st, eo, off, stats, status, C.byref(wall))
        out = []
        for i in range(count):
            if status[i]:
                out.append(None)
                continue
            a, b = voff[i], voff[i] + Vs[i]
            out.append(Placement(dev[a:b], st[a:b], eo[a:b], off[eoff[i]:eoff[i] + ns[i] + 1],
                                 stats[3 * i:3 * i + 3]))
        return status, out, wall.value

    @staticmethod
    def _text(call):
        """Two-phase string result: call(buf, buflen, needed_ptr) -> rc."""
        need = C.c_int64(0)
        rc = call(None, 0, C.byref(need))
        if need.value <= 0:
            return rc, ""
        buf = C.create_string_buffer(need.value)
        rc = call(buf, need.value, C.byref(need))
        return rc, buf.value.decode("utf-8")

    @classmethod
    def simulate_trace_csv(cls, rg, caps, cm, mem_mode, device_of, exec_order, exec_off):
        """simulate(record_trace) + trace_to_csv -> (csv text, event count)."""
        caps = _a(caps, np.int64)
        err = C.create_string_buffer(_ERRLEN)
        ev = C.c_int64()
        args = (_a(device_of, np.int32), _a(exec_order, np.int32), _a(exec_off, np.int32))
        rc, text = cls._text(lambda b, bl, nd: cls.lib().ref_simulate_trace_csv(
            rg.h, len(caps), caps, cm[0], cm[1], cm[2], mem_mode, *args, b, bl, nd, C.byref(ev), err, _ERRLEN))
        if rc:
            raise OracleError(rc, err.value.decode())
        return text, ev.value

    @classmethod
    def graph_json_roundtrip(cls, text: str) -> str:
        """parse_graph(text) -> graph_to_json."""
        raw = text.encode("utf-8")
        err = C.create_string_buffer(_ERRLEN)
        rc, out = cls._text(lambda b, bl, nd: cls.lib().ref_graph_json_roundtrip(raw, len(raw), b, bl, nd, err,
                                                                                 _ERRLEN))
        if rc:
            raise OracleError(rc, err.value.decode())
        return out

    @classmethod
    def graph_to_json(cls, rg) -> str:
        return cls._text(lambda b, bl, nd: cls.lib().ref_graph_to_json(rg.h, b, bl, nd))[1]

    @classmethod
    def comm_model_roundtrip(cls, text: str):
        """parse_comm_model(text) -> ((ic, pb, mode), save_comm_model text)."""
        raw = text.encode("utf-8")
        err = C.create_string_buffer(_ERRLEN)
        ic, pb, md = C.c_double(), C.c_double(), C.c_int32()
        rc, out = cls._text(lambda b, bl, nd: cls.lib().ref_comm_model_roundtrip(
            raw, len(raw), C.byref(ic), C.byref(pb), C.byref(md), b, bl, nd, err, _ERRLEN))
        if rc:
            raise OracleError(rc, err.value.decode())
        return (ic.value, pb.value, md.value), out

    @classmethod
    def placement_to_json(cls, rg, algorithm, device_of, exec_order, exec_off, sim_start, makespan, peaks) -> str:
        off = _a(exec_off, np.int32)
        args = (_a(device_of, np.int32), _a(exec_order, np.int32), off, _a(sim_start, np.int64), int(makespan),
                _a(peaks, np.int64))
        return cls._text(lambda b, bl, nd: cls.lib().ref_placement_to_json(
            rg.h, algorithm.encode(), len(off) - 1, *args, b, bl, nd))[1]

    @classmethod
    def placement_from_json(cls, rg, text: str, n: int):
        V = rg.sizes()[2]
        raw = text.encode("utf-8")
        algo = C.create_string_buffer(256)
        dev, st = np.zeros(max(V, 1), np.int32), np.zeros(max(V, 1), np.int64)
        eo, off = np.zeros(max(V, 1), np.int32), np.zeros(n + 1, np.int32)
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().ref_placement_from_json(rg.h, raw, len(raw), n, algo, 256, dev, st, eo, off, err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return algo.value.decode(), Placement(dev[:V], st[:V], eo[:V], off)

    # ---- graphs ----------------------------------------------------------
    class Graph:
        def __init__(self, handle):
            self.h = handle

        def __del__(self):
            if getattr(self, "h", None) and Ref._lib is not None:
                Ref._lib.ref_graph_free(self.h)
                self.h = None

        def sizes(self):
            vals = [C.c_int32() for _ in range(5)]
            Ref.lib().ref_graph_sizes(self.h, *[C.byref(v) for v in vals])
            return [v.value for v in vals]

        def meta(self):
            bv, be, V, E, mt = self.sizes()
            k, temp, perm, out = (np.zeros(V, np.int64) for _ in range(4))
            esrc, edst, ecount = (np.zeros(E, np.int32) for _ in range(3))
            ebytes = np.zeros(E, np.int64)
            group_of = np.zeros(bv, np.int32)
            members = np.zeros(max(mt, 1), np.int32)
            member_off = np.zeros(V + 1, np.int32)
            Ref.lib().ref_graph_meta(self.h, k, temp, perm, out, esrc, edst, ebytes, ecount,
                                     group_of, members, member_off)
            base_id = np.zeros(bv, np.int64)
            bs, bd = np.zeros(be, np.int32), np.zeros(be, np.int32)
            bb = np.zeros(be, np.int64)
            Ref.lib().ref_graph_base(self.h, base_id, bs, bd, bb)
            first_id = np.array([base_id[members[member_off[i]]] for i in range(V)], np.int64)
            return dict(V=V, E=E, k=k, temp=temp, perm=perm, out=out, esrc=esrc, edst=edst,
                        ebytes=ebytes, ecount=ecount, group_of=group_of,
                        members=members[:mt], member_off=member_off, first_id=first_id,
                        base_id=base_id)

    @classmethod
    def graph(cls, g: dict, pipeline: int = 1) -> "Ref.Graph":
        """pipeline: -1 singleton groups; else colocation + bit1 coplacement + bit2 fusion."""
        L = cls.lib()
        n = len(g["id"])
        e = len(g["src"])
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRLEN)
        rc = L.ref_graph_new(n, _a(g["id"], np.int64), _a(g["k"], np.int64),
                             _a(g["temp"], np.int64), _a(g["perm"], np.int64),
                             _a(g["out"], np.int64), _a(g["coloc"], np.int32),
                             _a(g["has_pair"], np.uint8), _a(g["pair"], np.int64), e,
                             _a(g["src"], np.int64), _a(g["dst"], np.int64),
                             _a(g["bytes"], np.int64), pipeline, C.byref(h), err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return cls.Graph(h)

    @classmethod
    def topo_order(cls, rg):
        V = rg.sizes()[2]
        order = np.zeros(max(V, 1), np.int32)
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().ref_meta_topo_order(rg.h, order, err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return order[:V]

    @classmethod
    def comm_time(cls, intercept, per_byte, nbytes):
        out = C.c_int64()
        err = C.create_string_buffer(256)
        rc = cls.lib().ref_comm_time(intercept, per_byte, int(nbytes), C.byref(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out.value

    @classmethod
    def bench_capacity(cls, rg, n, factor):
        return cls.lib().ref_bench_capacity(rg.h, n, factor)

    @classmethod
    def oracle_makespan(cls, rg, n, cm, capacity=None, mem_mode=1, max_nodes=12, max_devices=3,
                        max_extensions=200000):
        """oracle_makespan (oracle.cpp:185-212)."""
        out = C.c_int64()
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().ref_oracle_makespan(rg.h, n, cm[0], cm[1], cm[2], -1 if capacity is None else capacity,
                                           mem_mode, max_nodes, max_devices, max_extensions, C.byref(out), err,
                                           _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out.value

    @classmethod
    def critical_path(cls, rg):
        return cls.lib().ref_critical_path(rg.h)

    @classmethod
    def place(cls, rg, algo, caps, cm, fav=None):
        """algo 0/1/2 = m-topo/m-etf/m-sct; cm = (intercept, per_byte, mode 0 seq 1 par)."""
        V = rg.sizes()[2]
        caps = _a(caps, np.int64)
        n = len(caps)
        dev = np.zeros(max(V, 1), np.int32)
        st = np.zeros(max(V, 1), np.int64)
        eo = np.zeros(max(V, 1), np.int32)
        off = np.zeros(n + 1, np.int32)
        stats = np.zeros(3, np.int64)
        wall = C.c_int64()
        err = C.create_string_buffer(_ERRLEN)
        favp = None
        if fav is not None:
            favp = _a(fav, np.int32)
        rc = cls.lib().ref_place(rg.h, algo, n, caps, cm[0], cm[1], cm[2],
                                 favp.ctypes.data if favp is not None else None, dev, st, eo,
                                 off, stats, C.byref(wall), err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return Placement(dev[:V], st[:V], eo[:V], off, stats, wall.value)

    @classmethod
    def place_timed(cls, rg, algo, caps, cm, reps, fav=None):
        caps = _a(caps, np.int64)
        ns = np.zeros(reps, np.int64)
        err = C.create_string_buffer(_ERRLEN)
        favp = _opt(fav, np.int32)
        rc = cls.lib().ref_place_timed(rg.h, algo, len(caps), caps, cm[0], cm[1], cm[2],
                                       favp.ctypes.data if favp is not None else None, reps, ns,
                                       err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return ns

    @classmethod
    def place_batch(cls, graphs, algos, ns, caps2d, cm, threads=0):
        count = len(graphs)
        arr = (C.c_void_p * count)(*[g.h for g in graphs])
        status = np.zeros(count, np.int32)
        chk = np.zeros(count, np.int64)
        wall = C.c_int64()
        caps2d = _a(caps2d, np.int64)
        cls.lib().ref_place_batch(count, arr, _a(algos, np.int32), _a(ns, np.int32), caps2d,
                                  caps2d.shape[1], cm[0], cm[1], cm[2], threads, status, chk,
                                  C.byref(wall))
        return status, chk, wall.value

    @classmethod
    def schedulable_time(cls, rg, n, cm, dev_free, tail, device_of, finish, cache, j, p):
        out = C.c_int64()
        err = C.create_string_buffer(1024)
        rc = cls.lib().ref_schedulable_time(rg.h, n, cm[2], cm[0], cm[1], _a(dev_free, np.int64),
                                            _a(tail, np.int64), _a(device_of, np.int32),
                                            _a(finish, np.int64), _a(cache, np.int64), j, p,
                                            C.byref(out), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out.value

    @classmethod
    def simulate(cls, rg, caps, cm, mem_mode, device_of, exec_order, exec_off):
        V = rg.sizes()[2]
        caps = _a(caps, np.int64)
        n = len(caps)
        mk = C.c_int64()
        st = np.zeros(max(V, 1), np.int64)
        dev3n = np.zeros(3 * n, np.int64)
        x4 = np.zeros(4, np.int64)
        wall = C.c_int64()
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().ref_simulate(rg.h, n, caps, cm[0], cm[1], cm[2], mem_mode,
                                    _a(device_of, np.int32), _a(exec_order, np.int32),
                                    _a(exec_off, np.int32), C.byref(mk), st, dev3n, x4,
                                    C.byref(wall), err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return SimResult(mk.value, st[:V], dev3n, x4, wall.value)

    @classmethod
    def generate(cls, family, node_count, seed, branching=3, layers=4, edge_prob=0.3,
                 ranges=None, colocate_edge_frac=0.0, coplace_frac=0.0) -> dict:
        """Reference generate_graph; family 'branchy' | 'layered-chain' | 'random-dag'."""
        fam = {"branchy": 0, "layered-chain": 1, "random-dag": 2}[family]
        L = cls.lib()
        nn, ne = C.c_int32(), C.c_int32()
        err = C.create_string_buffer(1024)
        rng = _opt(ranges, np.int64)
        rp = rng.ctypes.data if rng is not None else None
        args0 = (fam, node_count, branching, layers, edge_prob, seed, rp, colocate_edge_frac,
                 coplace_frac)
        nulls = [None] * 11
        rc = L.ref_generate(*args0, 0, 0, C.byref(nn), C.byref(ne), *nulls, err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        N, M = nn.value, ne.value
        out = dict(id=np.zeros(N, np.int64), k=np.zeros(N, np.int64), temp=np.zeros(N, np.int64),
                   perm=np.zeros(N, np.int64), out=np.zeros(N, np.int64),
                   coloc=np.zeros(N, np.int32), has_pair=np.zeros(N, np.uint8),
                   pair=np.zeros(N, np.int64), src=np.zeros(M, np.int64),
                   dst=np.zeros(M, np.int64), bytes=np.zeros(M, np.int64))
        keys = ["id", "k", "temp", "perm", "out", "coloc", "has_pair", "pair", "src", "dst",
                "bytes"]
        rc = L.ref_generate(*args0, N, M, C.byref(nn), C.byref(ne),
                            *[out[k].ctypes.data for k in keys], err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out


# --------------------------------------------------------------------------
class _RsGraph(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int32), ("k", C.c_void_p), ("temp", C.c_void_p),
                ("perm", C.c_void_p), ("out", C.c_void_p), ("esrc", C.c_void_p),
                ("edst", C.c_void_p), ("ebytes", C.c_void_p), ("first_id", C.c_void_p)]


class Restate:
    """The plain-C restatement (oracle/restate.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(RESTATE_SO):
                build(ref=False)
            L = C.CDLL(RESTATE_SO)
            gp = C.POINTER(_RsGraph)
            cp, ip = C.c_char_p, C.c_int
            L.rs_comm_time.argtypes = [C.c_double, C.c_double, C.c_int64, C.POINTER(C.c_int)]
            L.rs_comm_time.restype = C.c_int64
            L.rs_place.argtypes = [gp, C.c_int32, C.c_int32, _i64p, C.c_double, C.c_double,
                                   C.c_int32, C.c_void_p, _i32p, _i64p, _i32p, _i32p, _i64p, cp,
                                   ip]
            L.rs_simulate.argtypes = [gp, C.c_int32, _i64p, C.c_double, C.c_double, C.c_int32,
                                      C.c_int32, _i32p, _i32p, _i32p, C.POINTER(C.c_int64), _i64p,
                                      _i64p, _i64p, cp, ip]
            L.rs_round_extract.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _f64p, C.c_double,
                                           _i32p, _i32p, _i32p, cp, ip]
            L.rs_topo_order.argtypes = [gp, _i32p, cp, ip]
            cls._lib = L
        return cls._lib

    @staticmethod
    def _g(m: dict):
        keep = {k: _a(m[k], np.int64) for k in ("k", "temp", "perm", "out", "ebytes")}
        keep["esrc"] = _a(m["esrc"], np.int32)
        keep["edst"] = _a(m["edst"], np.int32)
        fid = m.get("first_id")
        keep["first_id"] = None if fid is None else _a(fid, np.int64)
        g = _RsGraph(len(keep["k"]), len(keep["esrc"]), keep["k"].ctypes.data,
                     keep["temp"].ctypes.data, keep["perm"].ctypes.data,
                     keep["out"].ctypes.data, keep["esrc"].ctypes.data,
                     keep["edst"].ctypes.data, keep["ebytes"].ctypes.data,
                     keep["first_id"].ctypes.data if keep["first_id"] is not None else None)
        return g, keep

    @classmethod
    def comm_time(cls, intercept, per_byte, nbytes):
        err = C.c_int()
        v = cls.lib().rs_comm_time(intercept, per_byte, int(nbytes), C.byref(err))
        if err.value:
            raise OracleError(err.value, "comm_time: negative byte count")
        return v

    @classmethod
    def place(cls, m, algo, caps, cm, fav=None):
        g, keep = cls._g(m)
        V = g.V
        caps = _a(caps, np.int64)
        n = len(caps)
        dev = np.zeros(max(V, 1), np.int32)
        st = np.zeros(max(V, 1), np.int64)
        eo = np.zeros(max(V, 1), np.int32)
        off = np.zeros(n + 1, np.int32)
        stats = np.zeros(3, np.int64)
        err = C.create_string_buffer(_ERRLEN)
        favp = _opt(fav, np.int32)
        rc = cls.lib().rs_place(C.byref(g), algo, n, caps, cm[0], cm[1], cm[2],
                                favp.ctypes.data if favp is not None else None, dev, st, eo, off,
                                stats, err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return Placement(dev[:V], st[:V], eo[:V], off, stats)

    @classmethod
    def simulate(cls, m, caps, cm, mem_mode, device_of, exec_order, exec_off):
        g, keep = cls._g(m)
        V = g.V
        caps = _a(caps, np.int64)
        n = len(caps)
        mk = C.c_int64()
        st = np.zeros(max(V, 1), np.int64)
        dev3n = np.zeros(3 * n, np.int64)
        x4 = np.zeros(4, np.int64)
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().rs_simulate(C.byref(g), n, caps, cm[0], cm[1], cm[2], mem_mode,
                                   _a(device_of, np.int32), _a(exec_order, np.int32),
                                   _a(exec_off, np.int32), C.byref(mk), st, dev3n, x4, err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return SimResult(mk.value, st[:V], dev3n, x4)

    @classmethod
    def round_extract(cls, V, esrc, edst, x, threshold=0.1):
        fc = np.zeros(max(V, 1), np.int32)
        fp = np.zeros(max(V, 1), np.int32)
        s2 = np.zeros(2, np.int32)
        err = C.create_string_buffer(1024)
        esrc = _a(esrc, np.int32)
        rc = cls.lib().rs_round_extract(V, len(esrc), esrc, _a(edst, np.int32),
                                        _a(x, np.float64), threshold, fc, fp, s2, err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        return fc[:V], fp[:V], s2

    @classmethod
    def topo_order(cls, m):
        g, keep = cls._g(m)
        order = np.zeros(max(g.V, 1), np.int32)
        err = C.create_string_buffer(_ERRLEN)
        rc = cls.lib().rs_topo_order(C.byref(g), order, err, _ERRLEN)
        if rc:
            raise OracleError(rc, err.value.decode())
        return order[:g.V]
