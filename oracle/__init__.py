"""ctypes loader for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  The product path (paper_2507_21276_b200) never
imports, links or executes anything under oracle/.

The oracle itself is plain C (oracle/lemix_oracle.c), written from PAPER.md
Algorithm 1 and Eq. 1-4; see its header for the citations.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblemix_oracle.so")

LEMIX, RR, SEPARATE, FIXED, MIXLUF = 0, 1, 2, 3, 4
OK, EINVAL, EQCAP, EBUDGET = 0, 1, 6, 7


class Profile(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int32), ("n_stages", ctypes.c_int32),
                ("eta_f", ctypes.c_void_p), ("eta_b", ctypes.c_void_p), ("eta_d", ctypes.c_void_p)]


class Params(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("deprioritize", ctypes.c_int32),
                ("slo_mode", ctypes.c_int32), ("qcap", ctypes.c_int32),
                ("lambda1", ctypes.c_double), ("lambda2", ctypes.c_double), ("tau", ctypes.c_double),
                ("slo_mult", ctypes.c_double), ("slo_const", ctypes.c_double),
                ("sigma_floor", ctypes.c_double), ("lc0", ctypes.c_double), ("alpha", ctypes.c_double),
                ("mem_enable", ctypes.c_int32), ("mem_pad", ctypes.c_int32), ("mem_cap", ctypes.c_int64),
                ("mem_dt", ctypes.c_double), ("mem_tmax", ctypes.c_double), ("mem_pen", ctypes.c_double),
                ("sync_interval", ctypes.c_int32), ("sync_pad", ctypes.c_int32), ("sync_latency", ctypes.c_double),
                ("sep_dynamic", ctypes.c_int32), ("sep_pad", ctypes.c_int32), ("dyn_rate", ctypes.c_double),
                ("dyn_window", ctypes.c_double), ("cb_cmax", ctypes.c_int32), ("eq4_mode", ctypes.c_int32),
                ("cb_tw", ctypes.c_double), ("luf_delay", ctypes.c_double)]


SUMMARY_INT = ("n_tasks", "n_inf", "n_train", "n_slo_met", "n_deferrals", "active_nodes",
               "sum_version", "status", "n_mem_wait", "n_offload", "n_batches", "n_tbt")
SUMMARY_F64 = ("makespan", "throughput", "sum_ttft", "mean_ttft", "slo_attainment", "mean_util",
               "mean_len_std", "sum_tbt", "mean_tbt")


class Summary(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in SUMMARY_INT] + [(k, ctypes.c_double) for k in SUMMARY_F64]


COUNTERS = ("decisions", "alg1_calls", "stage_iters", "scan_consumed", "scan_break", "offset_adds",
            "lc_exp", "lc_cold", "commits_train", "eq4_checks", "deferrals", "version_scan", "max_qlen")


class Counters(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in COUNTERS]


SUMMARY_DTYPE = np.dtype([(k, np.int64) for k in SUMMARY_INT] + [(k, np.float64) for k in SUMMARY_F64])


_libs = {}


def _load(textbook: bool = False):
    """The oracle library; textbook=True loads the variant built with
    -DORC_TEXTBOOK (SURVEY.md 8c.4's division / Horner forms of Eq. 2), used
    only by tests/test_oracle_forms.py."""

    path = _LIB_PATH.replace(".so", "_textbook.so") if textbook else _LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        lib.orc_run_trace.restype = ctypes.c_int
        lib.orc_run_trace.argtypes = [ctypes.POINTER(Profile), ctypes.POINTER(Params), ctypes.c_int64,
                                      ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      ctypes.POINTER(Summary), ctypes.POINTER(Counters)]
        lib.orc_run_batch.restype = ctypes.c_int
        lib.orc_run_batch.argtypes = [ctypes.POINTER(Profile), ctypes.POINTER(Params), ctypes.c_int64,
                                      vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(Counters)]
        lib.orc_exp_neg.restype = ctypes.c_double
        lib.orc_exp_neg.argtypes = [ctypes.c_double]
        _libs[path] = lib
    return _libs[path]


@dataclass
class OracleParams:
    policy: int = LEMIX
    lambda1: float = 1.0
    lambda2: float = 1.0
    tau: float = 0.0
    slo_mult: float = 5.0
    sigma_floor: float = 1.0
    lc0: float = 0.0
    alpha: float = 0.5
    deprioritize: int = 1
    slo_mode: int = 0
    qcap: int = 512
    slo_const: float = 0.0
    # Algorithm 2 (NEXT-1, DESIGN.md R-mem); mem_enable = 0: unlimited memory
    mem_enable: int = 0
    mem_cap: int = 0
    mem_dt: float = 0.0
    mem_tmax: float = 0.0
    mem_pen: float = 0.0
    # Separate's checkpoint synchronisation (NEXT-3, DESIGN.md R-sync); 0 = off
    sync_interval: int = 0
    sync_latency: float = 0.0
    # SeparateDynamic (NEXT-3, DESIGN.md R-sepdyn); 0 = static alpha partition
    sep_dynamic: int = 0
    dyn_rate: float = 50.0
    dyn_window: float = 10.0
    # Algorithm 3 continuous batching (NEXT-2, DESIGN.md R-cb); 0 = off
    cb_cmax: int = 0
    cb_tw: float = 0.0
    # Eq. 4 reading (R-14 / R-14b)
    eq4_mode: int = 0
    # Mix-LUF scheduler latency per decision (DESIGN.md R-luf)
    luf_delay: float = 0.0

    def _c(self) -> Params:
        return Params(self.policy, self.deprioritize, self.slo_mode, self.qcap, self.lambda1,
                      self.lambda2, self.tau, self.slo_mult, self.slo_const, self.sigma_floor,
                      self.lc0, self.alpha, self.mem_enable, 0, self.mem_cap, self.mem_dt, self.mem_tmax,
                      self.mem_pen, self.sync_interval, 0, self.sync_latency, self.sep_dynamic, 0, self.dyn_rate,
                      self.dyn_window, self.cb_cmax, self.eq4_mode, self.cb_tw, self.luf_delay)


def _ptr(a):
    return None if a is None else a.ctypes.data


def exp_neg(t: float, textbook: bool = False) -> float:
    return _load(textbook).orc_exp_neg(float(t))


def _eta_d(eta_d):
    return None if eta_d is None else np.ascontiguousarray(eta_d, np.float64)


def run_trace(eta_f, eta_b, n_nodes, n_stages, arrival, lbk, n_inf, params: OracleParams,
              fixed_node=None, want_paths=False, want_cand=False, out_len=None, eta_d=None):
    """Run one trace; returns a dict of per-task outputs, summary, counters.
    out_len / eta_d: output tokens per task and decode cost table (continuous
    batching only)."""
    lib = _load()
    eta_f = np.ascontiguousarray(eta_f, np.float64)
    eta_b = np.ascontiguousarray(eta_b, np.float64)
    eta_d = _eta_d(eta_d)
    arrival = np.ascontiguousarray(arrival, np.float64)
    lbk = np.ascontiguousarray(lbk, np.uint32)
    out_len = None if out_len is None else np.ascontiguousarray(out_len, np.uint32)
    m = len(arrival)
    prof = Profile(n_nodes, n_stages, eta_f.ctypes.data, eta_b.ctypes.data, _ptr(eta_d))
    par = params._c()
    node_defer = np.zeros(m, np.uint32)
    dec = np.full(m, -1, np.int32)
    comp = np.zeros(m, np.float64)
    sf1 = np.zeros(m, np.float64)
    paths = np.zeros(m * n_stages * 4, np.float64) if want_paths else None
    cand = np.full(max(m, 1) * n_nodes * 3, np.nan) if want_cand else None
    fixed = None if fixed_node is None else np.ascontiguousarray(fixed_node, np.int32)
    sm = Summary()
    ct = Counters()
    st = lib.orc_run_trace(ctypes.byref(prof), ctypes.byref(par), m, int(n_inf), arrival.ctypes.data,
                           lbk.ctypes.data, _ptr(out_len), _ptr(fixed), node_defer.ctypes.data, dec.ctypes.data,
                           comp.ctypes.data, sf1.ctypes.data, _ptr(paths), _ptr(cand), ctypes.byref(sm),
                           ctypes.byref(ct))
    out = dict(status=st, node=(node_defer & 0xFFFF).astype(np.int32), defer=(node_defer >> 16).astype(np.int32),
               node_defer=node_defer, decision_idx=dec, completion=comp, start_f1=sf1,
               summary={k: getattr(sm, k) for k in SUMMARY_INT + SUMMARY_F64},
               counters={k: getattr(ct, k) for k in COUNTERS})
    if want_paths:
        out["paths"] = paths.reshape(m, n_stages, 4)
    if want_cand:
        out["cand"] = cand.reshape(max(m, 1), n_nodes, 3)[:m]
    return out


def run_batch(eta_f, eta_b, n_nodes, n_stages, traces, params: OracleParams, fixed_node=None,
              outputs=True, textbook=False, eta_d=None):
    """Run a CSR batch (workload.Traces; its out_len is passed when continuous
    batching is on).  Returns (summaries structured array, per-task dict or
    None, counters dict, first error status)."""
    lib = _load(textbook)
    eta_f = np.ascontiguousarray(eta_f, np.float64)
    eta_b = np.ascontiguousarray(eta_b, np.float64)
    eta_d = _eta_d(eta_d)
    prof = Profile(n_nodes, n_stages, eta_f.ctypes.data, eta_b.ctypes.data, _ptr(eta_d))
    out_len = (np.ascontiguousarray(traces.out_len, np.uint32)
               if params.cb_cmax > 0 and traces.out_len is not None else None)
    par = params._c()
    m = traces.n_tasks
    T = traces.n_traces
    sums = np.zeros(T, SUMMARY_DTYPE)
    ct = Counters()
    node_defer = np.zeros(m, np.uint32) if outputs else None
    dec = np.full(m, -1, np.int32) if outputs else None
    comp = np.zeros(m, np.float64) if outputs else None
    sf1 = np.zeros(m, np.float64) if outputs else None
    fixed = None if fixed_node is None else np.ascontiguousarray(fixed_node, np.int32)
    offsets = np.ascontiguousarray(traces.offsets, np.int64)
    n_inf = np.ascontiguousarray(traces.n_inf, np.int32)
    arrival = np.ascontiguousarray(traces.arrival, np.float64)
    lbk = np.ascontiguousarray(traces.lbk, np.uint32)
    st = lib.orc_run_batch(ctypes.byref(prof), ctypes.byref(par), T, offsets.ctypes.data,
                           n_inf.ctypes.data, arrival.ctypes.data, lbk.ctypes.data, _ptr(out_len), _ptr(fixed),
                           _ptr(node_defer), _ptr(dec), _ptr(comp), _ptr(sf1), sums.ctypes.data,
                           ctypes.byref(ct))
    per_task = None
    if outputs:
        per_task = dict(node_defer=node_defer, decision_idx=dec, completion=comp, start_f1=sf1)
    return sums, per_task, {k: getattr(ct, k) for k in COUNTERS}, st
