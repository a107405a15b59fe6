"""baechi-b200 — B200-native Baechi placement engine (arXiv 2301.08695).

Python face of the C ABI in ``include/baechi_b200.h`` (``libbaechi_b200.so``,
built in-tree for sm_100a). Names and error behaviour mirror the reference
C++ placer API (``/root/reference/proj/include/dagsched``):

=====================  ==============================================
reference              here
=====================  ==============================================
``place_mtopo``        :func:`place_mtopo`  (placers.hpp:73-74)
``place_metf``         :func:`place_metf`   (placers.hpp:78-79)
``place_msct``         :func:`place_msct`   (placers.hpp:87-89)
``simulate``           :func:`simulate`     (simulator.hpp:53-55)
``verify_placement``   :func:`verify_placement` (simulator.hpp:64-67)
``round_and_extract``  :func:`round_and_extract` (lp.hpp:88-90)
``comm_time``          :func:`comm_time`    (cost_model.hpp:29)
``schedulable_time``   :func:`schedulable_time` (placers.hpp:66-67)
``critical_path_us``   :func:`critical_path_us` (simulator.hpp:69)
``trace_to_csv``       :func:`trace_to_csv` (simulator.hpp:71)
``parse_comm_model``   :func:`parse_comm_model` / ``load_comm_model`` / ``save_comm_model``
``parse_graph``        :func:`parse_graph` / ``load_graph`` / :func:`graph_to_json`
``placement_to_json``  :func:`placement_to_json` / :func:`placement_from_json`
``max_comm_time``      :func:`max_comm_time` (cost_model.hpp:71)
``ValidationError``..  same names (errors.hpp:10-51)
=====================  ==============================================

Every compute call runs on the GPU through the .so; there is no CPU path.
If the library is missing or no CUDA device is visible the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbaechi_b200.so")

BX_OK, BX_VALIDATION, BX_INFEASIBLE, BX_SOLVER, BX_RUNTIME = 0, 2, 3, 4, 5
ALGOS = {"m-topo": 0, "m-etf": 1, "m-sct": 2}
SEQUENTIAL, PARALLEL = 0, 1
GRAPH_STATIC, TRAINING_PERSISTENT = 0, 1


# ---- errors (errors.hpp:10-51) ------------------------------------------
class Error(RuntimeError):
    kind = None

    def __init__(self, msg: str):
        super().__init__(msg)
        self.msg = msg


class ValidationError(Error):
    kind = BX_VALIDATION


class CycleError(ValidationError):
    pass


class InfeasibleError(Error):
    kind = BX_INFEASIBLE


class SolverError(Error):
    kind = BX_SOLVER


class DeviceError(Error):
    """CUDA/runtime failure (no reference analogue)."""
    kind = BX_RUNTIME


def _raise(status: int, msg: str):
    if status == BX_OK:
        return
    if status == BX_VALIDATION:
        if msg.startswith("meta graph is cyclic"):
            raise CycleError(msg)
        raise ValidationError(msg)
    if status == BX_INFEASIBLE:
        raise InfeasibleError(msg)
    if status == BX_SOLVER:
        raise SolverError(msg)
    raise DeviceError(msg)


# ---- ctypes mirror of baechi_b200.h ---------------------------------------
_vp = C.c_void_p


class _Graph(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int32),
                ("compute_us", _vp), ("temp_bytes", _vp), ("perm_bytes", _vp), ("out_bytes", _vp),
                ("esrc", _vp), ("edst", _vp), ("tensor_bytes", _vp),
                ("in_off", _vp), ("in_edge", _vp), ("out_off", _vp), ("first_id", _vp)]


class _BaseGraph(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("id", _vp), ("compute_us", _vp), ("temp_bytes", _vp),
                ("perm_bytes", _vp), ("out_bytes", _vp), ("coloc_label", _vp), ("has_pair", _vp),
                ("coplace_peer", _vp), ("edges", C.c_int32), ("src", _vp), ("dst", _vp),
                ("tensor_bytes", _vp)]


class _Grouping(C.Structure):
    _fields_ = [("base_nodes", C.c_int32), ("base_ids", _vp), ("group_of", _vp), ("members", _vp),
                ("member_off", _vp), ("edge_base_count", _vp)]


class _LpInfo(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("rel_gap", C.c_double), ("w", C.c_double),
                ("num_rows", C.c_int32), ("completion_rows", C.c_int32), ("precedence_rows", C.c_int32),
                ("child_rows", C.c_int32), ("parent_rows", C.c_int32), ("bound_rows", C.c_int32),
                ("host_ms", C.c_double), ("device_ms", C.c_double), ("factor_nnz", C.c_int64),
                ("update_pairs", C.c_int64)]


class _Comm(C.Structure):
    _fields_ = [("intercept_us", C.c_double), ("us_per_byte", C.c_double), ("mode", C.c_int32)]


class _Job(C.Structure):
    _fields_ = [("graph", C.c_int32), ("algo", C.c_int32), ("n", C.c_int32), ("capacity", _vp),
                ("cm", _Comm), ("fav_child", _vp), ("fav_len", C.c_int32)]


class _PlanOptions(C.Structure):
    _fields_ = [("no_small_frontier", C.c_int32), ("wide_min_vn", C.c_int32), ("wide_max_jobs", C.c_int32),
                ("list_len", C.c_int32), ("profile", C.c_int32), ("sim_heap_cap", C.c_int32),
                ("sim_trace", C.c_int32)]


class _PlacerState(C.Structure):
    _fields_ = [("V", C.c_int32), ("n", C.c_int32), ("mode", C.c_int32), ("dev_free", _vp), ("xfer_tail", _vp),
                ("device_of", _vp), ("finish_us", _vp), ("cache_arrival", _vp)]


class _TraceEvent(C.Structure):
    _fields_ = [("time_us", C.c_int64), ("device", C.c_int32), ("event", C.c_int32), ("node", C.c_int64)]


def _options(opts):
    """bx_plan_options from a dict (keys = field names); None = defaults."""
    o = _PlanOptions(0, -1, 0, 0, 0, -1, 0)
    for k, v in (opts or {}).items():
        if k not in dict(_PlanOptions._fields_):
            raise ValueError(f"unknown plan option {k!r}")
        setattr(o, k, int(v))
    return o


class _Placement(C.Structure):
    _fields_ = [("device_of", _vp), ("start_us", _vp), ("exec_order", _vp), ("exec_off", _vp),
                ("stats", C.c_int64 * 3), ("status", C.c_int32), ("msg", C.c_char * 256)]


class _SimReport(C.Structure):
    _fields_ = [("makespan_us", C.c_int64), ("start_us", _vp), ("peak_bytes", _vp), ("busy_us", _vp),
                ("idle_us", _vp), ("transfer_count", C.c_int64), ("transfer_bytes", C.c_int64),
                ("duplicate_transfers", C.c_int64), ("cache_hits", C.c_int64),
                ("status", C.c_int32), ("msg", C.c_char * 256)]


_lib = None


def lib():
    """Loads libbaechi_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(the placement engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        i32, i64, cp = C.c_int32, C.c_int64, C.c_char_p
        L.bx_version.restype = C.c_char_p
        L.bx_last_error.restype = C.c_char_p
        L.bx_last_message.restype = C.c_char_p
        L.bx_oracle_makespan.argtypes = [C.POINTER(_Graph), i32, C.POINTER(_Comm), i64, i32, i32, i32, i64,
                                         C.POINTER(i64), cp, C.c_int]
        L.bx_plan_message.argtypes = [_vp, i32, C.c_char_p, i64]
        L.bx_plan_message.restype = i64
        L.bx_device_count.restype = C.c_int
        L.bx_comm_time.argtypes = [C.POINTER(_Comm), i64, C.POINTER(i64)]
        L.bx_build_adjacency.argtypes = [i32, i32, _vp, _vp, _vp, _vp, _vp, cp, C.c_int]
        L.bx_plan_create.argtypes = [i32, C.POINTER(_Graph), i32, C.POINTER(_Job), i32,
                                     C.POINTER(_vp), cp, C.c_int]
        L.bx_plan_create_ex.argtypes = [i32, C.POINTER(_Graph), i32, C.POINTER(_Job), i32,
                                        C.POINTER(_PlanOptions), C.POINTER(_vp), cp, C.c_int]
        L.bx_plan_destroy.argtypes = [_vp]
        L.bx_plan_destroy.restype = None
        L.bx_plan_upload.argtypes = [_vp, _vp]
        L.bx_plan_place.argtypes = [_vp, _vp]
        L.bx_plan_download.argtypes = [_vp, _vp, C.POINTER(_Placement)]
        L.bx_plan_download_async.argtypes = [_vp, _vp]
        L.bx_plan_result_view.argtypes = [_vp, i32, C.POINTER(_Placement)]
        L.bx_plan_launch_count.argtypes = [_vp]
        L.bx_plan_job_kernel.argtypes = [_vp, i32]
        L.bx_simulate_ex.argtypes = [C.POINTER(_Graph), i32, _vp, C.POINTER(_Comm), i32, _vp, _vp, _vp,
                                     C.POINTER(_PlanOptions), C.POINTER(_SimReport)]
        L.bx_plan_kernel_ms.argtypes = [_vp]
        L.bx_plan_kernel_ms.restype = C.c_float
        L.bx_plan_kernel_times.argtypes = [_vp, i32, _vp]
        L.bx_plan_output_region.argtypes = [_vp, C.POINTER(_vp), C.POINTER(i64)]
        L.bx_plan_job_outputs.argtypes = [_vp, i32, _vp]
        L.bx_plan_profile.argtypes = [_vp, i32, _vp]
        L.bx_plan_simulate.argtypes = [_vp, i32, _vp]
        L.bx_plan_sim_download.argtypes = [_vp, _vp, C.POINTER(_SimReport)]
        L.bx_place.argtypes = [C.POINTER(_Graph), C.POINTER(_Job), C.POINTER(_Placement)]
        L.bx_simulate.argtypes = [C.POINTER(_Graph), i32, _vp, C.POINTER(_Comm), i32, _vp, _vp, _vp,
                                  C.POINTER(_SimReport)]
        L.bx_grouped_create.argtypes = [C.POINTER(_BaseGraph), i32, C.POINTER(_vp), cp, C.c_int]
        L.bx_grouped_view.argtypes = [_vp, C.POINTER(_Graph), C.POINTER(_Grouping)]
        L.bx_grouped_destroy.argtypes = [_vp]
        L.bx_grouped_destroy.restype = None
        L.bx_lp_solve.argtypes = [C.POINTER(_Graph), C.POINTER(_Comm), C.c_double, _vp, _vp,
                                   C.POINTER(_LpInfo), cp, C.c_int]
        L.bx_round_extract.argtypes = [i32, i32, _vp, _vp, _vp, C.c_double, _vp, _vp, _vp, cp, C.c_int]
        i64p = C.POINTER(i64)
        L.bx_schedulable_time.argtypes = [C.POINTER(_Graph), C.POINTER(_Comm), C.POINTER(_PlacerState), i32, _vp,
                                          _vp, _vp, cp, C.c_int]
        L.bx_critical_path_us.argtypes = [C.POINTER(_Graph), i64p, cp, C.c_int]
        L.bx_simulate_trace.argtypes = [C.POINTER(_Graph), i32, _vp, C.POINTER(_Comm), i32, _vp, _vp, _vp,
                                        C.POINTER(_SimReport), _vp, i64, i64p]
        L.bx_plan_sim_trace.argtypes = [_vp, i32, _vp, i64, i64p]
        L.bx_trace_to_csv.argtypes = [_vp, i64, _vp, i64, i64p]
        L.bx_comm_model_parse.argtypes = [cp, i64, C.POINTER(_Comm), cp, C.c_int]
        L.bx_comm_model_load.argtypes = [cp, C.POINTER(_Comm), cp, C.c_int]
        L.bx_comm_model_to_json.argtypes = [C.POINTER(_Comm), _vp, i64, i64p]
        L.bx_graph_parse.argtypes = [cp, i64, C.POINTER(_vp), cp, C.c_int]
        L.bx_graph_load.argtypes = [cp, C.POINTER(_vp), cp, C.c_int]
        L.bx_json_graph_view.argtypes = [_vp, C.POINTER(_BaseGraph), C.POINTER(_vp), C.POINTER(_vp),
                                         C.POINTER(i32)]
        L.bx_json_graph_destroy.argtypes = [_vp]
        L.bx_json_graph_destroy.restype = None
        L.bx_graph_to_json.argtypes = [C.POINTER(_BaseGraph), _vp, _vp, _vp, i64, i64p]
        L.bx_placement_to_json.argtypes = [C.POINTER(_Grouping), cp, i32, _vp, _vp, _vp, i64, _vp, _vp, i64, i64p]
        L.bx_placement_from_json.argtypes = [C.POINTER(_Grouping), i32, cp, i64, i32, cp, C.c_int, _vp, _vp, _vp,
                                             _vp, cp, C.c_int]
        L.bx_graph_save_bin.argtypes = [C.POINTER(_Graph), cp, cp, C.c_int]
        L.bx_graph_load_bin.argtypes = [cp, C.POINTER(_vp), C.POINTER(_Graph), cp, C.c_int]
        L.bx_bin_graph_destroy.argtypes = [_vp]
        L.bx_bin_graph_destroy.restype = None
        _lib = L
    return _lib


EXPORTED = ["bx_version", "bx_last_error", "bx_last_message", "bx_plan_message", "bx_oracle_makespan", "bx_device_count", "bx_comm_time", "bx_build_adjacency", "bx_plan_create",
            "bx_plan_create_ex", "bx_plan_job_kernel", "bx_simulate_ex",
            "bx_plan_destroy", "bx_plan_upload", "bx_plan_place", "bx_plan_download", "bx_plan_download_async", "bx_plan_result_view",
            "bx_plan_launch_count", "bx_plan_kernel_ms", "bx_plan_kernel_times",
            "bx_plan_output_region", "bx_plan_job_outputs", "bx_plan_profile", "bx_plan_simulate", "bx_plan_sim_download", "bx_place",
            "bx_simulate", "bx_round_extract", "bx_grouped_create", "bx_grouped_view", "bx_grouped_destroy", "bx_lp_solve",
            "bx_schedulable_time", "bx_critical_path_us", "bx_simulate_trace", "bx_plan_sim_trace", "bx_trace_to_csv",
            "bx_comm_model_parse", "bx_comm_model_load", "bx_comm_model_to_json", "bx_graph_parse", "bx_graph_load",
            "bx_json_graph_view", "bx_json_graph_destroy", "bx_graph_to_json", "bx_placement_to_json",
            "bx_placement_from_json", "bx_graph_save_bin", "bx_graph_load_bin", "bx_bin_graph_destroy"]


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


# ---- data model -----------------------------------------------------------
@dataclass
class CommModel:
    """CommModel (cost_model.hpp:19-24); mode 0 sequential, 1 parallel."""
    intercept_us: float = 0.0
    us_per_byte: float = 0.0
    mode: int = SEQUENTIAL

    def _c(self):
        return _Comm(float(self.intercept_us), float(self.us_per_byte), int(self.mode))


class MetaGraph:
    """A GroupedGraph (transforms.hpp:34-53) as flat arrays: meta-node
    aggregates, meta edges sorted by (src, dst), and the adjacency."""

    def __init__(self, k, temp, perm, out, esrc, edst, ebytes, first_id=None):
        self.k = _c(k, np.int64)
        self.temp = _c(temp, np.int64)
        self.perm = _c(perm, np.int64)
        self.out = _c(out, np.int64)
        self.esrc = _c(esrc, np.int32)
        self.edst = _c(edst, np.int32)
        self.ebytes = _c(ebytes, np.int64)
        self.first_id = None if first_id is None else _c(first_id, np.int64)
        self.V = len(self.k)
        self.E = len(self.esrc)
        self.in_off = np.zeros(self.V + 1, np.int32)
        self.out_off = np.zeros(self.V + 1, np.int32)
        self.in_edge = np.zeros(max(self.E, 1), np.int32)
        msg = C.create_string_buffer(256)
        rc = lib().bx_build_adjacency(self.V, self.E, _ptr(self.esrc), _ptr(self.edst),
                                      _ptr(self.in_off), _ptr(self.in_edge), _ptr(self.out_off), msg, 256)
        _raise(rc, msg.value.decode())

    @classmethod
    def from_dict(cls, m: dict) -> "MetaGraph":
        return cls(m["k"], m["temp"], m["perm"], m["out"], m["esrc"], m["edst"], m["ebytes"],
                   m.get("first_id"))

    def need(self):
        return self.perm + self.out + self.temp

    def _c(self):
        return _Graph(self.V, self.E, _ptr(self.k), _ptr(self.temp), _ptr(self.perm), _ptr(self.out),
                      _ptr(self.esrc), _ptr(self.edst), _ptr(self.ebytes), _ptr(self.in_off),
                      _ptr(self.in_edge), _ptr(self.out_off), _ptr(self.first_id))


@dataclass
class Placement:
    """Placement (placers.hpp:25-32) + PlacerStats (:34-38)."""
    algorithm: str
    device_of: np.ndarray
    start_us: np.ndarray
    exec_order_flat: np.ndarray
    exec_off: np.ndarray
    stats: tuple = (0, 0, 0)

    @property
    def exec_order(self):
        return [self.exec_order_flat[self.exec_off[d]:self.exec_off[d + 1]].tolist()
                for d in range(len(self.exec_off) - 1)]

    def __eq__(self, o):
        return (self.algorithm == o.algorithm and np.array_equal(self.device_of, o.device_of)
                and np.array_equal(self.start_us, o.start_us)
                and np.array_equal(self.exec_order_flat, o.exec_order_flat)
                and np.array_equal(self.exec_off, o.exec_off))


@dataclass
class TraceEvent:
    """TraceEvent (simulator.hpp:18-23)."""
    time_us: int
    device: int
    event: str  # start | finish | xfer_begin | xfer_end
    node: int


TRACE_EVENTS = ("start", "finish", "xfer_begin", "xfer_end")


@dataclass
class SimReport:
    """SimReport (simulator.hpp:25-34)."""
    makespan_us: int
    start_us: np.ndarray
    peak_bytes: np.ndarray
    busy_us: np.ndarray
    idle_us: np.ndarray
    transfer_count: int
    transfer_bytes: int
    duplicate_transfers: int
    cache_hits: int
    trace: list = field(default_factory=list)


@dataclass
class Job:
    graph: int
    algo: str
    capacity: np.ndarray
    cm: CommModel
    fav_child: np.ndarray | None = None


class Plan:
    """A device-resident batch of placement problems (bx_plan_*).

    ``upload`` copies host inputs to HBM, ``place`` runs K1+K2 on the given
    CUDA stream with inputs already resident, ``download`` copies the
    placements back (synchronising the stream)."""

    def __init__(self, graphs: list[MetaGraph], jobs: list[Job], device: int = 0, options: dict | None = None):
        """``options``: bx_plan_options fields (kernel dispatch; results never
        depend on them)."""
        self.graphs = graphs
        self.jobs = jobs
        self._keep = []
        self._gc = (_Graph * len(graphs))(*[g._c() for g in graphs])
        jc = []
        for j in jobs:
            cap = _c(j.capacity, np.int64)
            fav = None if j.fav_child is None else _c(j.fav_child, np.int32)
            self._keep += [cap, fav]
            jc.append(_Job(j.graph, ALGOS[j.algo], len(cap), _ptr(cap), j.cm._c(), _ptr(fav),
                           0 if fav is None else len(fav)))
        self._jc = (_Job * len(jobs))(*jc)
        h = _vp()
        msg = C.create_string_buffer(512)
        self._opt = _options(options)
        rc = lib().bx_plan_create_ex(len(graphs), self._gc, len(jobs), self._jc, device, C.byref(self._opt),
                                     C.byref(h), msg, 512)
        _raise(rc, msg.value.decode())
        self.h = h
        self.out = (_Placement * len(jobs))()

    def close(self):
        if getattr(self, "h", None):
            lib().bx_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, stream=None):
        rc = lib().bx_plan_upload(self.h, stream)
        _raise(rc, "bx_plan_upload failed")

    def place(self, stream=None):
        rc = lib().bx_plan_place(self.h, stream)
        _raise(rc, "bx_plan_place failed: " + lib().bx_last_error().decode())

    def launch_count(self) -> int:
        return lib().bx_plan_launch_count(self.h)

    KERNELS = {-1: "none", 0: "m-topo", 1: "warp", 2: "rounds", 3: "cta-seq", 4: "small-frontier", 5: "seq-small"}

    def job_kernel(self, i: int) -> str:
        """Which kernel placed job i in the last place()."""
        return self.KERNELS[lib().bx_plan_job_kernel(self.h, i)]

    PROFILE_FIELDS = ("rescan", "argmin", "rekey", "discard", "commit", "remove", "ready", "rows", "cache",
                      "insert", "emit", "steps", "commits", "rescans", "total")

    def profile(self, i: int) -> dict:
        """Latency breakdown of job i (plan built with options={"profile": 1})."""
        out = np.zeros(16, np.int64)
        rc = lib().bx_plan_profile(self.h, i, _ptr(out))
        _raise(rc, "no profile: create the plan with options={'profile': 1}")
        return dict(zip(self.PROFILE_FIELDS, out.tolist()))

    def kernel_ms(self) -> float:
        """CUDA-event time of the placer kernel(s) of the last place()."""
        return float(lib().bx_plan_kernel_ms(self.h))

    def kernel_times(self, count: int) -> list:
        """Placer-kernel CUDA-event times of the last `count` place() calls
        (<= 64 kept), oldest first; no host sync between the places."""
        out = np.zeros(max(count, 1), np.float32)
        got = lib().bx_plan_kernel_times(self.h, count, _ptr(out))
        if got < 0:
            raise DeviceError("bx_plan_kernel_times failed")
        return out[:got].astype(float).tolist()

    def output_region(self) -> tuple[int, int]:
        """(device pointer, bytes) of every job's device-resident outputs."""
        p, n = _vp(), C.c_int64()
        lib().bx_plan_output_region(self.h, C.byref(p), C.byref(n))
        return int(p.value or 0), n.value

    def job_outputs(self, i: int) -> list:
        """Byte offsets of job i's device_of, start_us, exec_order, exec_off,
        stats and status record inside output_region()."""
        o = np.zeros(6, np.int64)
        lib().bx_plan_job_outputs(self.h, i, _ptr(o))
        return o.tolist()

    def download_async(self, stream=None):
        """The download's device->pinned-host copy, enqueued on `stream` only."""
        _raise(lib().bx_plan_download_async(self.h, stream), "bx_plan_download_async failed")

    def download(self, stream=None):
        """One device->pinned-host copy of every job's placement."""
        rc = lib().bx_plan_download(self.h, stream, None)
        _raise(rc, "bx_plan_download failed: " + lib().bx_last_error().decode())
        for i in range(len(self.jobs)):
            lib().bx_plan_result_view(self.h, i, C.byref(self.out[i]))

    def result(self, i: int, copy=True) -> Placement:
        """Placement of job i; raises the job's reference error."""
        o = self.out[i]
        _raise(o.status, o.msg.decode())
        j = self.jobs[i]
        V = self.graphs[j.graph].V
        n = len(j.capacity)

        def view(ptr, ctype, count):
            if count == 0:
                return np.zeros(0, np.int32 if ctype is C.c_int32 else np.int64)
            a = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,))
            return a.copy() if copy else a

        return Placement(j.algo, view(o.device_of, C.c_int32, V), view(o.start_us, C.c_int64, V),
                         view(o.exec_order, C.c_int32, V), view(o.exec_off, C.c_int32, n + 1), tuple(o.stats))

    def status(self, i: int) -> tuple[int, str]:
        st = self.out[i].status
        if not st:
            return st, ""
        full = lib().bx_plan_message(self.h, i, None, 0)  # msg[256] holds a prefix
        buf = C.create_string_buffer(int(full) + 1)
        lib().bx_plan_message(self.h, i, buf, full + 1)
        return st, buf.value.decode()

    def simulate(self, mem_mode=TRAINING_PERSISTENT, stream=None):
        rc = lib().bx_plan_simulate(self.h, mem_mode, stream)
        _raise(rc, "bx_plan_simulate failed")

    def sim_download(self, stream=None) -> list:
        reps = (_SimReport * len(self.jobs))()
        keep = []
        for i, j in enumerate(self.jobs):
            V = self.graphs[j.graph].V
            n = len(j.capacity)
            b = [np.zeros(max(V, 1), np.int64)] + [np.zeros(n, np.int64) for _ in range(3)]
            keep.append(b)
            reps[i].start_us, reps[i].peak_bytes = _ptr(b[0]), _ptr(b[1])
            reps[i].busy_us, reps[i].idle_us = _ptr(b[2]), _ptr(b[3])
        rc = lib().bx_plan_sim_download(self.h, stream, reps)
        _raise(rc, "bx_plan_sim_download failed")
        out = []
        for i, j in enumerate(self.jobs):
            r = reps[i]
            if r.status:
                out.append((r.status, r.msg.decode()))
                continue
            V = self.graphs[j.graph].V
            b = keep[i]
            out.append(SimReport(r.makespan_us, b[0][:V], b[1], b[2], b[3], r.transfer_count,
                                 r.transfer_bytes, r.duplicate_transfers, r.cache_hits))
        return out


# ---- ingest: make_graph + build_grouped (host C++, csrc/ingest.cpp) --------
PIPE_SINGLETON, PIPE_COLOCATION, PIPE_COPLACEMENT, PIPE_FUSION = -1, 0, 2, 4


def _arr(ptr, ctype, count, dt):
    if count == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,)).astype(dt, copy=True)


def build_grouped(base: dict, coplacement: bool = True, fusion: bool = True, singleton: bool = False):
    """make_graph (graph.cpp:99-194) + build_grouped (bench.cpp:43-49).

    `base` holds node arrays id, k, temp, perm, out, optional coloc (int
    label, -1 none), has_pair + pair (peer id), and edge arrays src, dst,
    bytes (node ids). Returns (MetaGraph, grouping dict with base_ids,
    group_of, members, member_off, edge_base_count). Raises the reference's
    ValidationError / CycleError texts."""
    n = len(base["id"])
    keep = {k: _c(base[k], np.int64) for k in ("id", "k", "temp", "perm", "out", "src", "dst", "bytes")}
    coloc = base.get("coloc")
    keep["coloc"] = None if coloc is None else _c(coloc, np.int32)
    hp = base.get("has_pair")
    keep["has_pair"] = None if hp is None else _c(hp, np.uint8)
    keep["pair"] = None if hp is None else _c(base["pair"], np.int64)
    g = _BaseGraph(n, _ptr(keep["id"]), _ptr(keep["k"]), _ptr(keep["temp"]), _ptr(keep["perm"]),
                   _ptr(keep["out"]), _ptr(keep["coloc"]), _ptr(keep["has_pair"]), _ptr(keep["pair"]),
                   len(keep["src"]), _ptr(keep["src"]), _ptr(keep["dst"]), _ptr(keep["bytes"]))
    pipe = PIPE_SINGLETON if singleton else (PIPE_COPLACEMENT if coplacement else 0) | (PIPE_FUSION if fusion else 0)
    h = _vp()
    msg = C.create_string_buffer(4096)
    rc = lib().bx_grouped_create(C.byref(g), pipe, C.byref(h), msg, 4096)
    _raise(rc, msg.value.decode())
    try:
        mg = _Graph()
        gp = _Grouping()
        lib().bx_grouped_view(h, C.byref(mg), C.byref(gp))
        V, E, B = mg.V, mg.E, gp.base_nodes
        i64, i32 = C.c_int64, C.c_int32
        meta = MetaGraph(_arr(mg.compute_us, i64, V, np.int64), _arr(mg.temp_bytes, i64, V, np.int64),
                         _arr(mg.perm_bytes, i64, V, np.int64), _arr(mg.out_bytes, i64, V, np.int64),
                         _arr(mg.esrc, i32, E, np.int32), _arr(mg.edst, i32, E, np.int32),
                         _arr(mg.tensor_bytes, i64, E, np.int64), _arr(mg.first_id, i64, V, np.int64))
        off = _arr(gp.member_off, i32, V + 1, np.int32)
        grouping = dict(base_ids=_arr(gp.base_ids, i64, B, np.int64), group_of=_arr(gp.group_of, i32, B, np.int32),
                        members=_arr(gp.members, i32, int(off[-1]) if V else 0, np.int32), member_off=off,
                        edge_base_count=_arr(gp.edge_base_count, i32, E, np.int32))
    finally:
        lib().bx_grouped_destroy(h)
    return meta, grouping


# ---- reference-shaped entry points ---------------------------------------
def _one(gg: MetaGraph, algo: str, capacity, cm: CommModel, fav=None, stats_out=None,
         options: dict | None = None) -> Placement:
    if options is not None:  # a one-job plan with explicit dispatch options
        plan = Plan([gg], [Job(0, algo, capacity, cm, fav)], options=options)
        try:
            plan.upload()
            plan.place()
            plan.download()
            st, msg = plan.status(0)
            _raise(st, msg)
            p = plan.result(0)
        finally:
            plan.close()
        if stats_out is not None:
            stats_out[:] = list(p.stats)
        return p
    cap = _c(capacity, np.int64)
    favc = None if fav is None else _c(fav, np.int32)
    job = _Job(0, ALGOS[algo], len(cap), _ptr(cap), cm._c(), _ptr(favc), 0 if favc is None else len(favc))
    V, n = gg.V, len(cap)
    bufs = (np.zeros(max(V, 1), np.int32), np.zeros(max(V, 1), np.int64), np.zeros(max(V, 1), np.int32),
            np.zeros(n + 1, np.int32))
    out = _Placement(_ptr(bufs[0]), _ptr(bufs[1]), _ptr(bufs[2]), _ptr(bufs[3]))
    g = gg._c()
    lib().bx_place(C.byref(g), C.byref(job), C.byref(out))
    if out.status:
        _raise(out.status, lib().bx_last_message().decode())  # the full text (msg[256] is a prefix)
    if stats_out is not None:
        stats_out[:] = list(out.stats)
    return Placement(algo, bufs[0][:V].copy(), bufs[1][:V].copy(), bufs[2][:V].copy(), bufs[3].copy(),
                     tuple(out.stats))


def place_mtopo(gg: MetaGraph, capacity, cm: CommModel) -> Placement:
    return _one(gg, "m-topo", capacity, cm)


def place_metf(gg: MetaGraph, capacity, cm: CommModel, stats_out=None) -> Placement:
    return _one(gg, "m-etf", capacity, cm, stats_out=stats_out)


def place_msct(gg: MetaGraph, capacity, cm: CommModel, fav_child=None, stats_out=None) -> Placement:
    return _one(gg, "m-sct", capacity, cm, fav=fav_child, stats_out=stats_out)


def simulate(gg: MetaGraph, placement: Placement, capacity, cm: CommModel,
             mem_mode: int = TRAINING_PERSISTENT, options: dict | None = None,
             record_trace: bool = False) -> SimReport:
    """simulate (simulator.hpp:53-55); record_trace = SimOptions::record_trace."""
    cap = _c(capacity, np.int64)
    n = len(cap)
    V = gg.V
    b = [np.zeros(max(V, 1), np.int64)] + [np.zeros(max(n, 1), np.int64) for _ in range(3)]
    rep = _SimReport(0, _ptr(b[0]), _ptr(b[1]), _ptr(b[2]), _ptr(b[3]))
    dev = _c(placement.device_of, np.int32)
    eo = _c(placement.exec_order_flat, np.int32)
    off = _c(placement.exec_off, np.int32)
    if len(off) != n + 1 or len(dev) != V:
        raise ValidationError("placement does not match graph or roster")
    g = gg._c()
    cmc = cm._c()
    opt = _options(options)
    trace = []
    if record_trace:
        cap_ev = 2 * V + 2 * gg.E + 4
        tb = (_TraceEvent * cap_ev)()
        tl = C.c_int64()
        lib().bx_simulate_trace(C.byref(g), n, _ptr(cap), C.byref(cmc), mem_mode, _ptr(dev), _ptr(eo), _ptr(off),
                                C.byref(rep), tb, cap_ev, C.byref(tl))
        trace = [TraceEvent(tb[i].time_us, tb[i].device, TRACE_EVENTS[tb[i].event], tb[i].node)
                 for i in range(min(tl.value, cap_ev))]
    else:
        lib().bx_simulate_ex(C.byref(g), n, _ptr(cap), C.byref(cmc), mem_mode, _ptr(dev), _ptr(eo), _ptr(off),
                             C.byref(opt), C.byref(rep))
    _raise(rep.status, rep.msg.decode())
    return SimReport(rep.makespan_us, b[0][:V].copy(), b[1][:n].copy(), b[2][:n].copy(), b[3][:n].copy(),
                     rep.transfer_count, rep.transfer_bytes, rep.duplicate_transfers, rep.cache_hits, trace)


def verify_placement(gg, placement, capacity, cm, mem_mode=TRAINING_PERSISTENT):
    """verify_placement (simulator.cpp:280-294): (pass, diagnostic, report)."""
    try:
        r = simulate(gg, placement, capacity, cm, mem_mode)
        return True, "ok", r
    except Error as e:
        if isinstance(e, DeviceError):
            raise
        return False, e.msg, None


def round_and_extract(V: int, esrc, edst, x, threshold: float = 0.1):
    """round_and_extract (lp.cpp:280-326) on the GPU (K3). Returns
    (fav_child, fav_parent, (favorite_edges, repaired_nodes))."""
    esrc, edst, x = _c(esrc, np.int32), _c(edst, np.int32), _c(x, np.float64)
    fc = np.zeros(max(V, 1), np.int32)
    fp = np.zeros(max(V, 1), np.int32)
    s2 = np.zeros(2, np.int32)
    msg = C.create_string_buffer(256)
    rc = lib().bx_round_extract(V, len(esrc), _ptr(esrc), _ptr(edst), _ptr(x), float(threshold), _ptr(fc),
                                _ptr(fp), _ptr(s2), msg, 256)
    _raise(rc, msg.value.decode())
    return fc[:V], fp[:V], (int(s2[0]), int(s2[1]))


@dataclass
class LpSolution:
    """LpSolution (lp.hpp:47-53) plus SctLp row-class counts."""
    x: np.ndarray
    s: np.ndarray
    w: float
    iterations: int
    rel_gap: float
    rows: dict


def solve_relaxed(gg: MetaGraph, cm: CommModel, tolerance: float = 1e-6) -> LpSolution:
    """build_lp + solve_relaxed (lp.cpp:14-278): the reference's Mehrotra IPM,
    normal equations factored on the GPU. Raises SolverError like the
    reference."""
    x = np.zeros(max(gg.E, 1), np.float64)
    s = np.zeros(max(gg.V, 1), np.float64)
    info = _LpInfo()
    msg = C.create_string_buffer(512)
    g = gg._c()
    cmc = cm._c()
    rc = lib().bx_lp_solve(C.byref(g), C.byref(cmc), float(tolerance), _ptr(x), _ptr(s), C.byref(info), msg, 512)
    _raise(rc, msg.value.decode())
    rows = dict(total=info.num_rows, completion=info.completion_rows, precedence=info.precedence_rows,
                child=info.child_rows, parent=info.parent_rows, bound=info.bound_rows)
    sol = LpSolution(x[:gg.E].copy(), s[:gg.V].copy(), info.w, info.iterations, info.rel_gap, rows)
    sol.solver = dict(host_ms=info.host_ms, device_ms=info.device_ms, factor_nnz=info.factor_nnz,
                      update_pairs=info.update_pairs)
    return sol


def sct_favorites(gg: MetaGraph, cm: CommModel, threshold: float = 0.1, tolerance: float = 1e-6):
    """The m-SCT front half of run_placer (bench.cpp:63-70): solve the LP,
    round at `threshold` and extract favourites (K3 on the GPU). Returns
    (fav_child, fav_parent, (favorite_edges, repaired_nodes), LpSolution)."""
    sol = solve_relaxed(gg, cm, tolerance)
    fc, fp, st = round_and_extract(gg.V, gg.esrc, gg.edst, sol.x, threshold)
    return fc, fp, st, sol


def run_msct(gg: MetaGraph, capacity, cm: CommModel, threshold: float = 0.1, stats_out=None):
    """run_placer(Algo::MSct) (bench.cpp:63-70): LP -> favourites -> place_msct."""
    fc, _, _, _ = sct_favorites(gg, cm, threshold)
    return place_msct(gg, capacity, cm, fc, stats_out=stats_out)


def comm_time(cm: CommModel, nbytes: int) -> int:
    out = C.c_int64()
    cmc = cm._c()
    rc = lib().bx_comm_time(C.byref(cmc), int(nbytes), C.byref(out))
    if rc:
        raise ValidationError("comm_time: negative byte count")
    return out.value


def max_comm_time(gg: MetaGraph, cm: CommModel) -> int:
    return max((comm_time(cm, b) for b in gg.ebytes.tolist()), default=0)


def device_count() -> int:
    return lib().bx_device_count()


# ---- partial-schedule queries (placers.hpp:49-67, simulator.hpp:69) --------
class PlacerState:
    """PlacerState (placers.hpp:49-60): dev_free / xfer_tail [n], device_of /
    finish_us [V], cache_arrival [V*n] (-1 absent); initialised as the
    reference's constructor does (placers.cpp:31-37)."""

    def __init__(self, meta_count: int, device_count: int, mode: int):
        self.mode = int(mode)
        self.dev_free = np.zeros(device_count, np.int64)
        self.xfer_tail = np.zeros(device_count, np.int64)
        self.device_of = np.full(meta_count, -1, np.int32)
        self.finish_us = np.zeros(meta_count, np.int64)
        self.cache_arrival = np.full(meta_count * device_count, -1, np.int64)

    def _c(self):
        self._keep = [_c(a, dt) for a, dt in ((self.dev_free, np.int64), (self.xfer_tail, np.int64),
                                              (self.device_of, np.int32), (self.finish_us, np.int64),
                                              (self.cache_arrival, np.int64))]
        k = self._keep
        return _PlacerState(len(k[2]), len(k[0]), self.mode, *[_ptr(a) for a in k])


def schedulable_times(st: PlacerState, nodes, devices, gg: MetaGraph, cm: CommModel) -> np.ndarray:
    """schedulable_time (placers.cpp:83-91) for every (nodes[i], devices[i]),
    evaluated on the GPU in one launch."""
    js, ps = _c(nodes, np.int32), _c(devices, np.int32)
    out = np.zeros(max(len(js), 1), np.int64)
    msg = C.create_string_buffer(512)
    g, cmc, sc = gg._c(), cm._c(), st._c()
    rc = lib().bx_schedulable_time(C.byref(g), C.byref(cmc), C.byref(sc), len(js), _ptr(js), _ptr(ps), _ptr(out),
                                   msg, 512)
    _raise(rc, msg.value.decode())
    return out[:len(js)]


def schedulable_time(st: PlacerState, j: int, p: int, gg: MetaGraph, cm: CommModel) -> int:
    """schedulable_time (placers.hpp:66-67): earliest start of j on p."""
    return int(schedulable_times(st, [j], [p], gg, cm)[0])


def critical_path_us(gg: MetaGraph) -> int:
    """critical_path_us (simulator.cpp:296-309) on the GPU."""
    out = C.c_int64()
    msg = C.create_string_buffer(4096)
    g = gg._c()
    rc = lib().bx_critical_path_us(C.byref(g), C.byref(out), msg, 4096)
    _raise(rc, msg.value.decode())
    return out.value


def oracle_makespan(gg: MetaGraph, device_count: int, cm: CommModel, capacity=None,
                    mode: int = TRAINING_PERSISTENT, max_nodes: int = 12, max_devices: int = 3,
                    max_extensions: int = 200000) -> int:
    """oracle_makespan (oracle.hpp:29-34): exact minimum makespan over every
    canonical device assignment and DAG-consistent execution order, each
    scored by the GPU simulator. Raises InfeasibleError like the reference
    (too large, nothing fits)."""
    out = C.c_int64()
    msg = C.create_string_buffer(4096)
    g = gg._c()
    cmc = cm._c()
    rc = lib().bx_oracle_makespan(C.byref(g), int(device_count), C.byref(cmc), -1 if capacity is None else int(capacity),
                                  int(mode), int(max_nodes), int(max_devices), int(max_extensions), C.byref(out),
                                  msg, 4096)
    _raise(rc, msg.value.decode())
    return out.value


def _text(call) -> tuple[int, str]:
    need = C.c_int64(0)
    call(None, 0, C.byref(need))
    buf = C.create_string_buffer(max(need.value, 1))
    rc = call(buf, need.value, C.byref(need))
    return rc, buf.value.decode("utf-8")


def trace_to_csv(trace: list) -> str:
    """trace_to_csv (simulator.cpp:311-324)."""
    arr = (_TraceEvent * max(len(trace), 1))()
    for i, ev in enumerate(trace):
        arr[i] = _TraceEvent(ev.time_us, ev.device, TRACE_EVENTS.index(ev.event), ev.node)
    return _text(lambda b, bl, nd: lib().bx_trace_to_csv(arr, len(trace), b, bl, nd))[1]


# ---- interchange IO (csrc/jsonio.cpp) -------------------------------------
def parse_comm_model(text: str) -> CommModel:
    """parse_comm_model (cost_model.cpp:71-111)."""
    raw = text.encode("utf-8")
    out = _Comm()
    msg = C.create_string_buffer(1024)
    rc = lib().bx_comm_model_parse(raw, len(raw), C.byref(out), msg, 1024)
    _raise(rc, msg.value.decode())
    return CommModel(out.intercept_us, out.us_per_byte, out.mode)


def load_comm_model(path: str) -> CommModel:
    """load_comm_model (cost_model.cpp:113-122), e.g. comm_model_test.json."""
    out = _Comm()
    msg = C.create_string_buffer(1024)
    rc = lib().bx_comm_model_load(os.fsencode(path), C.byref(out), msg, 1024)
    _raise(rc, msg.value.decode())
    return CommModel(out.intercept_us, out.us_per_byte, out.mode)


def comm_model_to_json(cm: CommModel) -> str:
    """The text save_comm_model writes (cost_model.cpp:124-134)."""
    c = cm._c()
    return _text(lambda b, bl, nd: lib().bx_comm_model_to_json(C.byref(c), b, bl, nd))[1]


def save_comm_model(cm: CommModel, path: str) -> None:
    with open(path, "w") as f:
        f.write(comm_model_to_json(cm))


class JsonGraph:
    """A parsed graph file (parse_graph, graph.cpp:196-272, before
    make_graph): ``base`` is the dict build_grouped takes, plus node names
    and colocation group strings."""

    def __init__(self, handle):
        self.h = handle
        bg = _BaseGraph()
        names, groups, ng = _vp(), _vp(), C.c_int32()
        lib().bx_json_graph_view(handle, C.byref(bg), C.byref(names), C.byref(groups), C.byref(ng))
        n, e = bg.nodes, bg.edges
        i64, i32, u8 = C.c_int64, C.c_int32, C.c_uint8
        self.base = dict(id=_arr(bg.id, i64, n, np.int64), k=_arr(bg.compute_us, i64, n, np.int64),
                         temp=_arr(bg.temp_bytes, i64, n, np.int64), perm=_arr(bg.perm_bytes, i64, n, np.int64),
                         out=_arr(bg.out_bytes, i64, n, np.int64), coloc=_arr(bg.coloc_label, i32, n, np.int32),
                         has_pair=_arr(bg.has_pair, u8, n, np.uint8),
                         pair=_arr(bg.coplace_peer, i64, n, np.int64), src=_arr(bg.src, i64, e, np.int64),
                         dst=_arr(bg.dst, i64, e, np.int64), bytes=_arr(bg.tensor_bytes, i64, e, np.int64))
        npp = C.cast(names, C.POINTER(C.c_char_p))
        gpp = C.cast(groups, C.POINTER(C.c_char_p))
        self.names = [npp[i].decode("utf-8") for i in range(n)]
        self.groups = [gpp[i].decode("utf-8") for i in range(ng.value)]
        lib().bx_json_graph_destroy(handle)
        self.h = None


def parse_graph(text: str) -> JsonGraph:
    """parse_graph (graph.cpp:196-262) up to make_graph (run by build_grouped)."""
    raw = text.encode("utf-8")
    h = _vp()
    msg = C.create_string_buffer(4096)
    rc = lib().bx_graph_parse(raw, len(raw), C.byref(h), msg, 4096)
    _raise(rc, msg.value.decode())
    return JsonGraph(h)


def load_graph(path: str) -> JsonGraph:
    h = _vp()
    msg = C.create_string_buffer(4096)
    rc = lib().bx_graph_load(os.fsencode(path), C.byref(h), msg, 4096)
    _raise(rc, msg.value.decode())
    return JsonGraph(h)


def graph_to_json(base: dict, names=None, groups=None) -> str:
    """graph_to_json (graph.cpp:283-309) of a base graph dict."""
    n = len(base["id"])
    keep = {k: _c(base[k], np.int64) for k in ("id", "k", "temp", "perm", "out", "src", "dst", "bytes")}
    coloc = base.get("coloc")
    keep["coloc"] = None if coloc is None else _c(coloc, np.int32)
    hp = base.get("has_pair")
    keep["has_pair"] = None if hp is None else _c(hp, np.uint8)
    keep["pair"] = None if hp is None else _c(base["pair"], np.int64)
    g = _BaseGraph(n, _ptr(keep["id"]), _ptr(keep["k"]), _ptr(keep["temp"]), _ptr(keep["perm"]),
                   _ptr(keep["out"]), _ptr(keep["coloc"]), _ptr(keep["has_pair"]), _ptr(keep["pair"]),
                   len(keep["src"]), _ptr(keep["src"]), _ptr(keep["dst"]), _ptr(keep["bytes"]))
    nm = None if names is None else (C.c_char_p * max(n, 1))(*[x.encode("utf-8") for x in names])
    gr = None if groups is None else (C.c_char_p * max(len(groups), 1))(*[x.encode("utf-8") for x in groups])
    return _text(lambda b, bl, nd: lib().bx_graph_to_json(C.byref(g), nm, gr, b, bl, nd))[1]


def _grouping_c(grouping: dict):
    keep = dict(base_ids=_c(grouping["base_ids"], np.int64), group_of=_c(grouping["group_of"], np.int32),
                members=_c(grouping["members"], np.int32), member_off=_c(grouping["member_off"], np.int32),
                edge_base_count=_c(grouping.get("edge_base_count", np.zeros(1)), np.int32))
    return _Grouping(len(keep["base_ids"]), _ptr(keep["base_ids"]), _ptr(keep["group_of"]), _ptr(keep["members"]),
                     _ptr(keep["member_off"]), _ptr(keep["edge_base_count"])), keep


def placement_to_json(grouping: dict, placement: Placement, report: SimReport) -> str:
    """placement_to_json (placers.cpp:367-386) with a simulated report."""
    gp, keep = _grouping_c(grouping)
    eo, off = _c(placement.exec_order_flat, np.int32), _c(placement.exec_off, np.int32)
    st, pk = _c(report.start_us, np.int64), _c(report.peak_bytes, np.int64)
    algo = placement.algorithm.encode("utf-8")
    return _text(lambda b, bl, nd: lib().bx_placement_to_json(C.byref(gp), algo, len(off) - 1, _ptr(eo), _ptr(off),
                                                              _ptr(st), int(report.makespan_us), _ptr(pk), b,
                                                              bl, nd))[1]


def placement_from_json(grouping: dict, V: int, text: str, device_count: int) -> Placement:
    """placement_from_json (placers.cpp:388-432)."""
    gp, keep = _grouping_c(grouping)
    raw = text.encode("utf-8")
    algo = C.create_string_buffer(256)
    dev, st = np.zeros(max(V, 1), np.int32), np.zeros(max(V, 1), np.int64)
    eo, off = np.zeros(max(V, 1), np.int32), np.zeros(device_count + 1, np.int32)
    msg = C.create_string_buffer(1024)
    rc = lib().bx_placement_from_json(C.byref(gp), V, raw, len(raw), device_count, algo, 256, _ptr(dev), _ptr(st),
                                      _ptr(eo), _ptr(off), msg, 1024)
    _raise(rc, msg.value.decode())
    return Placement(algo.value.decode(), dev[:V].copy(), st[:V].copy(), eo[:V].copy(), off.copy())


def save_graph_bin(gg: MetaGraph, path: str) -> None:
    """Binary CSR sidecar of a meta graph (csrc/jsonio.cpp)."""
    msg = C.create_string_buffer(1024)
    g = gg._c()
    rc = lib().bx_graph_save_bin(C.byref(g), os.fsencode(path), msg, 1024)
    _raise(rc, msg.value.decode())


def load_graph_bin(path: str) -> MetaGraph:
    h = _vp()
    v = _Graph()
    msg = C.create_string_buffer(1024)
    rc = lib().bx_graph_load_bin(os.fsencode(path), C.byref(h), C.byref(v), msg, 1024)
    _raise(rc, msg.value.decode())
    try:
        i64, i32 = C.c_int64, C.c_int32
        V, E = v.V, v.E
        return MetaGraph(_arr(v.compute_us, i64, V, np.int64), _arr(v.temp_bytes, i64, V, np.int64),
                         _arr(v.perm_bytes, i64, V, np.int64), _arr(v.out_bytes, i64, V, np.int64),
                         _arr(v.esrc, i32, E, np.int32), _arr(v.edst, i32, E, np.int32),
                         _arr(v.tensor_bytes, i64, E, np.int64),
                         None if not v.first_id else _arr(v.first_id, i64, V, np.int64))
    finally:
        lib().bx_bin_graph_destroy(h)
