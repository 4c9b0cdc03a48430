"""ctypes binding of liblemix.so (include/lemix.h) -- argument marshalling only.

Every step of the placement path runs in the CUDA kernels behind the C ABI;
this module only converts numpy arrays / torch tensors to pointers.  There is
no CPU fallback: if the shared library or a CUDA device is missing, calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LMX_LIB: developer override (A/B of alternative builds of the same sources)
LIB_PATH = os.environ.get("LMX_LIB") or os.path.join(_HERE, "liblemix.so")

LMX_OK, LMX_EINVAL, LMX_ESTATE, LMX_ENOMEM, LMX_ECUDA, LMX_ENCCL, LMX_EQCAP, LMX_EBUDGET, LMX_ETIMEOUT = range(9)
LMX_LEMIX, LMX_RR, LMX_SEPARATE, LMX_FIXED, LMX_MIXLUF = range(5)
LMX_HOST, LMX_DEVICE = 0, 1
STATUS_NAMES = {0: "LMX_OK", 1: "LMX_EINVAL", 2: "LMX_ESTATE", 3: "LMX_ENOMEM", 4: "LMX_ECUDA",
                5: "LMX_ENCCL", 6: "LMX_EQCAP", 7: "LMX_EBUDGET",
                8: "LMX_ETIMEOUT"}

EXPORTS = ("lmx_params_default", "lmx_create", "lmx_destroy", "lmx_last_error", "lmx_load_profile",
           "lmx_load_traces", "lmx_set_params", "lmx_set_cells", "lmx_set_cell_params", "lmx_set_outputs", "lmx_run", "lmx_sync",
           "lmx_get_assignments", "lmx_get_times", "lmx_get_candidates", "lmx_get_summaries", "lmx_get_cells",
           "lmx_allreduce_cells", "lmx_nccl_unique_id", "lmx_nccl_comm_init", "lmx_nccl_comm_destroy",
           "lmx_get_timing", "lmx_get_geometry")


class lmx_profile(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int32), ("n_stages", ctypes.c_int32),
                ("eta_f", ctypes.c_void_p), ("eta_b", ctypes.c_void_p), ("eta_d", ctypes.c_void_p)]


class lmx_traces(ctypes.Structure):
    _fields_ = [("n_traces", ctypes.c_int64), ("offsets", ctypes.c_void_p), ("n_inf", ctypes.c_void_p),
                ("arrival", ctypes.c_void_p), ("len_batch_kind", ctypes.c_void_p),
                ("fixed_node", ctypes.c_void_p), ("out_len", ctypes.c_void_p)]


class lmx_params(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("deprioritize", ctypes.c_int32), ("slo_mode", ctypes.c_int32),
                ("qcap", ctypes.c_int32), ("lambda1", ctypes.c_double), ("lambda2", ctypes.c_double),
                ("tau", ctypes.c_double), ("slo_mult", ctypes.c_double), ("slo_const", ctypes.c_double),
                ("sigma_floor", ctypes.c_double), ("lc0", ctypes.c_double), ("alpha", ctypes.c_double),
                ("mem_enable", ctypes.c_int32), ("mem_pad", ctypes.c_int32), ("mem_cap", ctypes.c_int64),
                ("mem_dt", ctypes.c_double), ("mem_tmax", ctypes.c_double), ("mem_pen", ctypes.c_double),
                ("sync_interval", ctypes.c_int32), ("sync_pad", ctypes.c_int32), ("sync_latency", ctypes.c_double),
                ("sep_dynamic", ctypes.c_int32), ("sep_pad", ctypes.c_int32), ("dyn_rate", ctypes.c_double),
                ("dyn_window", ctypes.c_double), ("debug_level", ctypes.c_int32), ("debug_pad", ctypes.c_int32),
                ("cb_cmax", ctypes.c_int32), ("eq4_mode", ctypes.c_int32), ("cb_tw", ctypes.c_double),
                ("luf_delay", ctypes.c_double)]


SUMMARY_INT = ("n_tasks", "n_inf", "n_train", "n_slo_met", "n_deferrals", "active_nodes", "sum_version",
               "status", "n_mem_wait", "n_offload", "n_batches", "n_tbt")
SUMMARY_F64 = ("makespan", "throughput", "sum_ttft", "mean_ttft", "slo_attainment", "mean_util",
               "mean_len_std", "sum_tbt", "mean_tbt")
SUMMARY_DTYPE = np.dtype([(k, np.int64) for k in SUMMARY_INT] + [(k, np.float64) for k in SUMMARY_F64])
CELL_INT = ("n_traces", "n_failed", "n_tasks", "n_inf", "n_train", "n_slo_met", "n_deferrals",
            "sum_active_nodes", "sum_version")
CELL_F64 = ("sum_makespan", "sum_throughput", "sum_ttft", "sum_mean_ttft", "sum_slo_attainment",
            "sum_mean_util", "sum_mean_len_std")
CELL_DTYPE = np.dtype([(k, np.int64) for k in CELL_INT] + [(k, np.float64) for k in CELL_F64])

_lib = None


def load_library():
    """Load liblemix.so or raise (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"liblemix.so not built ({LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
    sig = {
        "lmx_params_default": (None, [ctypes.POINTER(lmx_params)]),
        "lmx_create": (st, [ctypes.POINTER(vp), ctypes.c_int, vp]),
        "lmx_destroy": (None, [vp]),
        "lmx_last_error": (ctypes.c_char_p, [vp]),
        "lmx_load_profile": (st, [vp, ctypes.POINTER(lmx_profile)]),
        "lmx_load_traces": (st, [vp, ctypes.POINTER(lmx_traces), ctypes.c_int]),
        "lmx_set_params": (st, [vp, ctypes.POINTER(lmx_params)]),
        "lmx_set_cells": (st, [vp, vp, i32]),
        "lmx_set_cell_params": (st, [vp, i32, vp, vp, vp]),
        "lmx_set_outputs": (st, [vp, ctypes.c_int]),
        "lmx_run": (st, [vp]),
        "lmx_sync": (st, [vp]),
        "lmx_get_assignments": (st, [vp, vp, vp, ctypes.c_int]),
        "lmx_get_times": (st, [vp, vp, vp, ctypes.c_int]),
        "lmx_get_candidates": (st, [vp, vp, ctypes.c_int]),
        "lmx_get_summaries": (st, [vp, vp]),
        "lmx_get_cells": (st, [vp, vp]),
        "lmx_allreduce_cells": (st, [vp, vp]),
        "lmx_nccl_unique_id": (st, [vp]),
        "lmx_nccl_comm_init": (st, [ctypes.POINTER(vp), ctypes.c_int, vp, ctypes.c_int, ctypes.c_int]),
        "lmx_nccl_comm_destroy": (st, [vp]),
        "lmx_get_timing": (st, [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                                ctypes.POINTER(i32)]),
        "lmx_get_geometry": (st, [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                                  ctypes.POINTER(i32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class LemixError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    """Pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


@dataclass
class Params:
    policy: int = LMX_LEMIX
    deprioritize: int = 1
    slo_mode: int = 0
    qcap: int = 512
    lambda1: float = 1.0
    lambda2: float = 1.0
    tau: float = 0.0
    slo_mult: float = 5.0
    slo_const: float = 0.0
    sigma_floor: float = 1.0
    lc0: float = 0.0
    alpha: float = 0.5
    # Algorithm 2 memory model (include/lemix.h lmx_params.mem_*); 0 = unlimited memory
    mem_enable: int = 0
    mem_cap: int = 0
    mem_dt: float = 0.0
    mem_tmax: float = 0.0
    mem_pen: float = 0.0
    # Separate's checkpoint synchronisation (lmx_params.sync_*); 0 = co-located proxy
    sync_interval: int = 0
    sync_latency: float = 0.0
    # SeparateDynamic (lmx_params.sep_dynamic / dyn_rate / dyn_window)
    sep_dynamic: int = 0
    dyn_rate: float = 50.0
    dyn_window: float = 10.0
    # stepwise debug output (lmx_params.debug_level): 1 = (II, R, f) per decision and node
    debug_level: int = 0
    # Algorithm 3 continuous batching (lmx_params.cb_*); 0 = off
    cb_cmax: int = 0
    cb_tw: float = 0.0
    # Eq. 4 reading (0 = R-14, 1 = R-14b) and Mix-LUF's scheduler latency
    eq4_mode: int = 0
    luf_delay: float = 0.0

    def c(self) -> lmx_params:
        return lmx_params(self.policy, self.deprioritize, self.slo_mode, self.qcap, self.lambda1, self.lambda2,
                          self.tau, self.slo_mult, self.slo_const, self.sigma_floor, self.lc0, self.alpha,
                          self.mem_enable, 0, self.mem_cap, self.mem_dt, self.mem_tmax, self.mem_pen,
                          self.sync_interval, 0, self.sync_latency, self.sep_dynamic, 0, self.dyn_rate,
                          self.dyn_window, self.debug_level, 0, self.cb_cmax, self.eq4_mode, self.cb_tw,
                          self.luf_delay)


class Context:
    """One lmx_ctx (one GPU).  Methods mirror the C calls one to one."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        h = ctypes.c_void_p()
        st = self.lib.lmx_create(ctypes.byref(h), device, stream)
        if st != LMX_OK:
            raise LemixError(st, self.lib.lmx_last_error(None).decode())
        self.h = h
        self._keep = []   # host arrays that must outlive async copies

    def _check(self, st):
        if st != LMX_OK:
            raise LemixError(st, self.lib.lmx_last_error(self.h).decode())
        return st

    def close(self):
        if self.h:
            self.lib.lmx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lmx_load_profile(self, n_nodes, n_stages, eta_f, eta_b, eta_d=None):
        eta_f = np.ascontiguousarray(eta_f, np.float64)
        eta_b = np.ascontiguousarray(eta_b, np.float64)
        eta_d = None if eta_d is None else np.ascontiguousarray(eta_d, np.float64)
        pr = lmx_profile(n_nodes, n_stages, eta_f.ctypes.data, eta_b.ctypes.data, _ptr(eta_d))
        return self._check(self.lib.lmx_load_profile(self.h, ctypes.byref(pr)))

    def lmx_load_traces(self, offsets, n_inf, arrival, lbk, fixed_node=None, mem=LMX_HOST, out_len=None):
        offsets = np.ascontiguousarray(offsets, np.int64)
        n_inf = np.ascontiguousarray(n_inf, np.int32)
        self._keep = [offsets, n_inf, arrival, lbk, fixed_node, out_len]
        tr = lmx_traces(len(n_inf), offsets.ctypes.data, n_inf.ctypes.data, _ptr(arrival), _ptr(lbk),
                        _ptr(fixed_node), _ptr(out_len))
        return self._check(self.lib.lmx_load_traces(self.h, ctypes.byref(tr), mem))

    def lmx_set_params(self, params: Params):
        p = params.c()
        return self._check(self.lib.lmx_set_params(self.h, ctypes.byref(p)))

    def lmx_set_cells(self, cell_of_trace, n_cells):
        arr = None if cell_of_trace is None else np.ascontiguousarray(cell_of_trace, np.int32)
        return self._check(self.lib.lmx_set_cells(self.h, _ptr(arr), n_cells))

    def lmx_set_cell_params(self, n_cells, lambda1=None, lambda2=None, tau=None):
        arrs = [None if a is None else np.ascontiguousarray(a, np.float64) for a in (lambda1, lambda2, tau)]
        return self._check(self.lib.lmx_set_cell_params(self.h, n_cells, *[_ptr(a) for a in arrs]))

    def lmx_set_outputs(self, per_task: bool):
        return self._check(self.lib.lmx_set_outputs(self.h, 1 if per_task else 0))

    def lmx_run(self):
        return self._check(self.lib.lmx_run(self.h))

    def lmx_sync(self, raise_on_trace_error=False):
        st = self.lib.lmx_sync(self.h)
        if st in (LMX_ESTATE, LMX_ECUDA) or (st != LMX_OK and raise_on_trace_error):
            self._check(st)
        return st

    def last_error(self):
        return self.lib.lmx_last_error(self.h).decode()

    def lmx_get_assignments(self, node_defer=None, decision_idx=None, mem=LMX_HOST):
        return self._check(self.lib.lmx_get_assignments(self.h, _ptr(node_defer), _ptr(decision_idx), mem))

    def lmx_get_times(self, completion=None, start_f1=None, mem=LMX_HOST):
        return self._check(self.lib.lmx_get_times(self.h, _ptr(completion), _ptr(start_f1), mem))

    def lmx_get_candidates(self, cand, mem=LMX_HOST):
        return self._check(self.lib.lmx_get_candidates(self.h, _ptr(cand), mem))

    def lmx_get_summaries(self, n_traces):
        out = np.zeros(n_traces, SUMMARY_DTYPE)
        self._check(self.lib.lmx_get_summaries(self.h, out.ctypes.data))
        return out

    def lmx_get_cells(self, n_cells=1):
        out = np.zeros(n_cells, CELL_DTYPE)
        self._check(self.lib.lmx_get_cells(self.h, out.ctypes.data))
        return out

    def lmx_allreduce_cells(self, comm):
        return self._check(self.lib.lmx_allreduce_cells(self.h, comm))

    def lmx_get_timing(self):
        k, r, n = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32()
        self._check(self.lib.lmx_get_timing(self.h, ctypes.byref(k), ctypes.byref(r), ctypes.byref(n)))
        return k.value, r.value, n.value

    def lmx_get_geometry(self):
        v = [ctypes.c_int32() for _ in range(4)]
        self._check(self.lib.lmx_get_geometry(self.h, *[ctypes.byref(x) for x in v]))
        return tuple(x.value for x in v)


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.lmx_nccl_unique_id(buf)
    if st != LMX_OK:
        raise LemixError(st, "ncclGetUniqueId failed")
    return buf.raw


def nccl_comm_init(nranks: int, uid: bytes, rank: int, device: int):
    lib = load_library()
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    st = lib.lmx_nccl_comm_init(ctypes.byref(comm), nranks, buf, rank, device)
    if st != LMX_OK:
        raise LemixError(st, "ncclCommInitRank failed")
    return comm


def nccl_comm_destroy(comm):
    load_library().lmx_nccl_comm_destroy(comm)


@dataclass
class RunResult:
    status: int
    summaries: np.ndarray
    cells: np.ndarray
    node_defer: np.ndarray | None = None
    decision_idx: np.ndarray | None = None
    completion: np.ndarray | None = None
    start_f1: np.ndarray | None = None
    cand: np.ndarray | None = None
    kernel_ms: float = 0.0
    run_ms: float = 0.0
    launches: int = 0
    error: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def node(self):
        return None if self.node_defer is None else (self.node_defer & 0xFFFF).astype(np.int32)


def run(eta_f, eta_b, n_nodes, n_stages, traces, params: Params | None = None, device: int = 0,
        outputs: bool = True, fixed_node=None, cells=None, n_cells: int = 1, ctx: Context | None = None,
        cell_params: dict | None = None, eta_d=None):
    """Convenience: create -> load -> run -> sync -> fetch, all through the C ABI.
    `traces` is a workload.Traces (host arrays)."""
    params = params or Params()
    own = ctx is None
    ctx = ctx or Context(device)
    try:
        ctx.lmx_load_profile(n_nodes, n_stages, eta_f, eta_b, eta_d)
        out_len = (np.ascontiguousarray(traces.out_len, np.uint32)
                   if params.cb_cmax > 0 and traces.out_len is not None else None)
        ctx.lmx_load_traces(traces.offsets, traces.n_inf, np.ascontiguousarray(traces.arrival, np.float64),
                            np.ascontiguousarray(traces.lbk, np.uint32),
                            None if fixed_node is None else np.ascontiguousarray(fixed_node, np.int32),
                            out_len=out_len)
        ctx.lmx_set_params(params)
        ctx.lmx_set_cells(cells, n_cells)
        if cell_params is not None:   # {"lambda1": [...], "lambda2": [...], "tau": [...]} per cell
            ctx.lmx_set_cell_params(n_cells, **cell_params)
        ctx.lmx_set_outputs(outputs)
        ctx.lmx_run()
        st = ctx.lmx_sync()
        err = ctx.last_error() if st != LMX_OK else ""
        res = RunResult(status=st, summaries=ctx.lmx_get_summaries(traces.n_traces),
                        cells=ctx.lmx_get_cells(n_cells), error=err)
        if outputs:
            m = traces.n_tasks
            res.node_defer = np.zeros(m, np.uint32)
            res.decision_idx = np.zeros(m, np.int32)
            res.completion = np.zeros(m, np.float64)
            res.start_f1 = np.zeros(m, np.float64)
            ctx.lmx_get_assignments(res.node_defer, res.decision_idx)
            ctx.lmx_get_times(res.completion, res.start_f1)
        if params.debug_level == 1:
            res.cand = np.zeros((traces.n_tasks, n_nodes, 3), np.float64)
            ctx.lmx_get_candidates(res.cand)
        res.kernel_ms, res.run_ms, res.launches = ctx.lmx_get_timing()
        return res
    finally:
        if own:
            ctx.close()
