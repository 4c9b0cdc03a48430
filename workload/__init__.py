"""Seeded synthetic workload traces and profile tables.

This module is the ONE thing the oracle and the CUDA path share: it draws the
inputs (arrival times, lengths, batch sizes, the profile table) and holds none
of the scheduling method's arithmetic.  The sampling itself is C
(``workload/gen.c``, multi-threaded over traces, one xoshiro256** stream per
trace seeded by SplitMix64(seed_base + trace), so outputs do not depend on the
thread count).

Shapes:
  * arrivals: Poisson (exponential gaps) or a Gamma renewal
    process with CV = 3 ("bursty", LMSYS-shaped);
  * lengths: LogNormal, clamped to [16, 2048] (heavy right tail of
    HH-RLHF/SHP); inference median 64 / sigma_log 1.0, training
    median 128 / sigma_log 0.8, heterogeneous median 64 / sigma_log 1.5;
  * training: Poisson earliest-release times, or continuous retraining
    (a_min = 0), micro-batch C_train;
  * profile: Llama-8B row of Table 1: 0.11 s forward / 0.15 s
    backward per stage at C = 1, l = 500 -> eta_F = 4.4e-7, eta_B = 6.0e-7 at
    S = 2, scaled by 2/S for other stage counts.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libworkload.so")
_lib = None

L_BITS = 12
C_SHIFT = 12
KIND_SHIFT = 20


class _Spec(ctypes.Structure):
    _fields_ = [
        ("n_inf", ctypes.c_int64), ("n_train", ctypes.c_int64),
        ("arrival_kind", ctypes.c_int32), ("train_kind", ctypes.c_int32),
        ("rate_inf", ctypes.c_double), ("rate_train", ctypes.c_double), ("cv", ctypes.c_double),
        ("len_inf_median", ctypes.c_double), ("len_inf_sigma", ctypes.c_double),
        ("len_train_median", ctypes.c_double), ("len_train_sigma", ctypes.c_double),
        ("len_min", ctypes.c_int32), ("len_max", ctypes.c_int32),
        ("batch_inf", ctypes.c_int32), ("batch_train", ctypes.c_int32),
        ("out_median", ctypes.c_double), ("out_sigma", ctypes.c_double),
    ]


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.wl_generate.restype = ctypes.c_int
        _lib.wl_generate.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib.wl_generate_seeds.restype = ctypes.c_int
        _lib.wl_generate_seeds.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    return _lib


@dataclass(frozen=True)
class WorkloadSpec:
    n_inf: int
    n_train: int
    rate_inf: float = 10.0
    rate_train: float = 10.0
    bursty: bool = False
    cv: float = 3.0
    continuous_training: bool = False
    len_inf_median: float = 64.0
    len_inf_sigma: float = 1.0
    len_train_median: float = 128.0
    len_train_sigma: float = 0.8
    len_min: int = 16
    len_max: int = 2048
    batch_inf: int = 1
    batch_train: int = 1
    out_median: float = 200.0
    out_sigma: float = 1.0

    def _c(self) -> _Spec:
        return _Spec(self.n_inf, self.n_train, 1 if self.bursty else 0,
                     1 if self.continuous_training else 0, self.rate_inf, self.rate_train, self.cv,
                     self.len_inf_median, self.len_inf_sigma, self.len_train_median,
                     self.len_train_sigma, self.len_min, self.len_max, self.batch_inf,
                     self.batch_train, self.out_median, self.out_sigma)


@dataclass
class Traces:
    """CSR batch of traces: trace t owns tasks [offsets[t], offsets[t+1]); its
    first n_inf[t] tasks are inference (arrival order), the rest training."""
    offsets: np.ndarray   # int64 [T+1]
    n_inf: np.ndarray     # int32 [T]
    arrival: np.ndarray   # float64 [M]
    lbk: np.ndarray       # uint32 [M]
    out_len: np.ndarray   # uint32 [M]

    @property
    def n_traces(self) -> int:
        return len(self.n_inf)

    @property
    def n_tasks(self) -> int:
        return int(self.offsets[-1])

    def trace(self, t: int) -> "Traces":
        o0, o1 = int(self.offsets[t]), int(self.offsets[t + 1])
        return Traces(np.array([0, o1 - o0], np.int64), self.n_inf[t:t + 1].copy(),
                      self.arrival[o0:o1], self.lbk[o0:o1],
                      None if self.out_len is None else self.out_len[o0:o1])

    def subset(self, idx) -> "Traces":
        return concat([self.trace(int(t)) for t in idx])


def pack(length, batch, kind):
    length = np.asarray(length, np.uint32)
    batch = np.asarray(batch, np.uint32)
    kind = np.asarray(kind, np.uint32)
    return (length | (batch << C_SHIFT) | (kind << KIND_SHIFT)).astype(np.uint32)


def unpack(lbk):
    lbk = np.asarray(lbk, np.uint32)
    return lbk & 0xFFF, (lbk >> C_SHIFT) & 0xFF, (lbk >> KIND_SHIFT) & 1


def generate(spec: WorkloadSpec, n_traces: int, seed_base: int = 1, n_threads: int | None = None,
             out=None) -> Traces:
    """Generate n_traces traces of spec; trace t uses seed seed_base + t."""
    lib = _load()
    per = spec.n_inf + spec.n_train
    m = per * n_traces
    if out is None:
        arrival = np.empty(m, np.float64)
        lbk = np.empty(m, np.uint32)
        out_len = np.empty(m, np.uint32)
    else:
        arrival, lbk, out_len = out
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    rc = lib.wl_generate(ctypes.byref(spec._c()), n_traces, seed_base, arrival.ctypes.data,
                         lbk.ctypes.data, None if out_len is None else out_len.ctypes.data, n_threads)
    if rc != 0:
        raise ValueError(f"invalid workload spec: {spec}")
    offsets = np.arange(n_traces + 1, dtype=np.int64) * per
    n_inf = np.full(n_traces, spec.n_inf, np.int32)
    return Traces(offsets, n_inf, arrival, lbk, out_len)


def concat(parts) -> Traces:
    parts = list(parts)
    sizes = [p.n_tasks for p in parts]
    offsets = [np.zeros(1, np.int64)]
    base = 0
    for p, sz in zip(parts, sizes):
        offsets.append(p.offsets[1:] + base)
        base += sz
    return Traces(np.concatenate(offsets), np.concatenate([p.n_inf for p in parts]).astype(np.int32),
                  np.concatenate([p.arrival for p in parts]), np.concatenate([p.lbk for p in parts]),
                  None if any(p.out_len is None for p in parts) else np.concatenate([p.out_len for p in parts]))


def from_lists(traces) -> Traces:
    """Build a batch from python lists: each trace is a list of
    (arrival, length, batch, kind[, out_len]) with kind 0 = inference,
    1 = training, out_len = decode steps (default 0).  Tasks are stably
    partitioned (inference first); inference tasks must be in arrival order,
    training tasks in release order."""
    parts = []
    for tr in traces:
        inf = [t for t in tr if t[3] == 0]
        trn = [t for t in tr if t[3] == 1]
        rows = inf + trn
        arr = np.array([t[0] for t in rows], np.float64)
        lbk = pack([t[1] for t in rows], [t[2] for t in rows], [t[3] for t in rows]) if rows else \
            np.zeros(0, np.uint32)
        out = np.array([t[4] if len(t) > 4 else 0 for t in rows], np.uint32)
        parts.append(Traces(np.array([0, len(rows)], np.int64), np.array([len(inf)], np.int32), arr,
                            lbk, out))
    return concat(parts)


# --------------------------------------------------------------------------
# Profile tables (Table 1, tab:models, lines 749-754; reference shape
# C = 1, l = 500 is the SPEC.md:160 reading, eta = per-stage latency / 500^2).
# --------------------------------------------------------------------------
TABLE1 = {  # name: (forward s, backward s)
    "gpt-400m": (0.03, 0.04), "gpt-1.4b": (0.08, 0.09), "gpt-2.5b": (0.12, 0.14),
    "llama-8b": (0.11, 0.15), "llama-13b": (0.24, 0.36), "llama-70b": (0.73, 1.05),
}


def profile(n_nodes: int, n_stages: int, model: str = "llama-8b"):
    """Homogeneous (eta_f, eta_b) float64 [N*S] node-major tables."""
    fwd, bwd = TABLE1[model]
    scale = 2.0 / n_stages
    ef = fwd / 250000.0 * scale
    eb = bwd / 250000.0 * scale
    return (np.full(n_nodes * n_stages, ef, np.float64), np.full(n_nodes * n_stages, eb, np.float64))


def decode_profile(n_nodes: int, n_stages: int, model: str = "llama-8b"):
    """eta_D [N*S] (seconds per context token per item of one decode step on a
    stage GPU): one decode step of one request at the Table 1
    reference context (500 tokens) costs 1/200 of that shape's forward (0.55 ms
    per Llama-8B stage at S = 2), so a 200-token output over a ~100-token
    context keeps a stage busy ~0.1 s."""
    fwd, _ = TABLE1[model]
    return np.full(n_nodes * n_stages, fwd * (2.0 / n_stages) / 200.0 / 500.0, np.float64)


def batch_timeout(n_stages: int, model: str = "llama-8b", length: int = 64) -> float:
    """T_w = 0.5 x the inference latency of the median request
    (a `length`-token prompt, C = 1) through all stages: 0.5 * S * eta_F * l^2."""
    ef, _ = profile(1, n_stages, model)
    return 0.5 * float(ef[0]) * n_stages * length * length


# --------------------------------------------------------------------------
# The BASELINE.json configs (SURVEY.md §8d concrete inputs)
# --------------------------------------------------------------------------
def tiny_spec(rate=20.0, alpha=0.5, n_inf=200):
    n_train = int(round(n_inf * alpha / (1.0 - alpha)))
    return WorkloadSpec(n_inf=n_inf, n_train=n_train, rate_inf=rate * (1 - alpha), rate_train=rate * alpha)


def paper_spec(n_inf=20000, n_train=4000):
    return WorkloadSpec(n_inf=n_inf, n_train=n_train, rate_inf=50.0, bursty=True, cv=3.0,
                        continuous_training=True, batch_train=4)


def sweep_spec(rate, alpha=0.5, tasks=1000):
    n_train = int(round(tasks * alpha))
    return WorkloadSpec(n_inf=tasks - n_train, n_train=n_train, rate_inf=rate * (1 - alpha),
                        rate_train=rate * alpha)


SWEEP_RATES = tuple(float(10 * k) for k in range(1, 17))


def large_spec(rate=1600.0, alpha=0.5, n_inf=200000):
    n_train = int(round(n_inf * alpha / (1.0 - alpha)))
    return WorkloadSpec(n_inf=n_inf, n_train=n_train, rate_inf=rate * (1 - alpha),
                        rate_train=rate * alpha, len_inf_median=64.0, len_inf_sigma=1.5)


def mc_spec(bursty=False, n_inf=10000, n_train=10000, rate=50.0):
    return WorkloadSpec(n_inf=n_inf, n_train=n_train, rate_inf=rate / 2, rate_train=rate / 2,
                        bursty=bursty, cv=3.0)


def mc_traces(n_traces=65536, seed_base=1, n_inf=10000, n_train=10000, n_threads=None, out=None,
              with_out_len=True) -> Traces:
    """Monte Carlo config: the first half Poisson, the second half bursty
    (Gamma CV = 3), seeds seed_base + t.  `out` = (arrival, lbk) buffers to
    fill (e.g. pinned host memory)."""
    half = n_traces // 2
    per = n_inf + n_train
    m = per * n_traces
    if out is None:
        arrival = np.empty(m, np.float64)
        lbk = np.empty(m, np.uint32)
    else:
        arrival, lbk = out
    out_len = np.empty(m, np.uint32) if with_out_len else None
    ol = (lambda a, b: None) if out_len is None else (lambda a, b: out_len[a:b])
    generate(mc_spec(False, n_inf, n_train), half, seed_base, n_threads,
             out=(arrival[:half * per], lbk[:half * per], ol(0, half * per)))
    generate(mc_spec(True, n_inf, n_train), n_traces - half, seed_base + half, n_threads,
             out=(arrival[half * per:], lbk[half * per:], ol(half * per, m)))
    offsets = np.arange(n_traces + 1, dtype=np.int64) * per
    return Traces(offsets, np.full(n_traces, n_inf, np.int32), arrival, lbk, out_len)


def mc_traces_subset(idx, n_total=65536, seed_base=1, n_inf=10000, n_train=10000, n_threads=None, out=None,
                     with_out_len=True) -> Traces:
    """Traces idx (sorted indices into the n_total-trace Monte Carlo set of
    mc_traces(n_total, seed_base)): trace t is Poisson when t < n_total // 2,
    bursty otherwise, with seed seed_base + t -- the same arrays mc_traces
    would give for those indices (a rank's shard of the fixed seed set)."""
    idx = np.asarray(idx, np.int64)
    if idx.size and (np.any(np.diff(idx) <= 0) or idx[0] < 0 or idx[-1] >= n_total):
        raise ValueError("idx must be sorted, unique and in [0, n_total)")
    half = n_total // 2
    per = n_inf + n_train
    m = per * len(idx)
    if out is None:
        arrival = np.empty(m, np.float64)
        lbk = np.empty(m, np.uint32)
    else:
        arrival, lbk = out
    out_len = np.empty(m, np.uint32) if with_out_len else None
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    lib = _load()
    k = int(np.searchsorted(idx, half))
    for lo, hi, bursty in ((0, k, False), (k, len(idx), True)):
        if hi <= lo:
            continue
        seeds = np.ascontiguousarray(seed_base + idx[lo:hi], np.uint64)
        rc = lib.wl_generate_seeds(ctypes.byref(mc_spec(bursty, n_inf, n_train)._c()), hi - lo, seeds.ctypes.data,
                                   arrival[lo * per:].ctypes.data, lbk[lo * per:].ctypes.data,
                                   None if out_len is None else out_len[lo * per:].ctypes.data, n_threads)
        if rc != 0:
            raise ValueError("invalid workload spec")
    offsets = np.arange(len(idx) + 1, dtype=np.int64) * per
    return Traces(offsets, np.full(len(idx), n_inf, np.int32), arrival, lbk, out_len)


__all__ = ["mc_traces_subset", "decode_profile", "batch_timeout", "WorkloadSpec", "Traces", "generate", "concat", "from_lists", "pack", "unpack", "profile",
           "tiny_spec", "paper_spec", "sweep_spec", "large_spec", "mc_spec", "mc_traces", "SWEEP_RATES",
           "TABLE1", "replace"]
