"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle
import workload

INT_FIELDS = ("n_tasks", "n_inf", "n_train", "n_slo_met", "n_deferrals", "active_nodes", "sum_version", "status",
              "n_mem_wait", "n_offload", "n_batches", "n_tbt")
F64_FIELDS = ("makespan", "throughput", "sum_ttft", "mean_ttft", "slo_attainment", "mean_util", "mean_len_std",
              "sum_tbt", "mean_tbt")
REL_TOL = 1e-12   # north_star: fp summaries within 1e-12 relative


def oracle_params(lp) -> oracle.OracleParams:
    return oracle.OracleParams(policy=lp.policy, lambda1=lp.lambda1, lambda2=lp.lambda2, tau=lp.tau,
                               slo_mult=lp.slo_mult, sigma_floor=lp.sigma_floor, lc0=lp.lc0, alpha=lp.alpha,
                               deprioritize=lp.deprioritize, slo_mode=lp.slo_mode, qcap=lp.qcap,
                               slo_const=lp.slo_const, mem_enable=lp.mem_enable, mem_cap=lp.mem_cap,
                               mem_dt=lp.mem_dt, mem_tmax=lp.mem_tmax, mem_pen=lp.mem_pen,
                               sync_interval=lp.sync_interval, sync_latency=lp.sync_latency,
                               sep_dynamic=lp.sep_dynamic, dyn_rate=lp.dyn_rate, dyn_window=lp.dyn_window,
                               cb_cmax=lp.cb_cmax, cb_tw=lp.cb_tw, eq4_mode=lp.eq4_mode, luf_delay=lp.luf_delay)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.maximum(np.abs(a), np.abs(b))
    diff = np.abs(a - b)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(den > 0, diff / den, 0.0)
    r = np.where(a == b, 0.0, r)   # equal infinities
    return float(r.max()) if r.size else 0.0


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64))


def compare_summaries(gs, osum, ok_mask=None, bitwise=True):
    assert len(gs) == len(osum)
    for k in INT_FIELDS:
        g = gs[k]
        o = osum[k]
        bad = np.nonzero(g != o)[0]
        assert bad.size == 0, f"summary {k} differs at traces {bad[:8]}: gpu {g[bad[:8]]} oracle {o[bad[:8]]}"
    for k in F64_FIELDS:
        e = rel_err(gs[k], osum[k])
        assert e <= REL_TOL, f"summary {k} rel err {e}"
        if bitwise:
            assert bits_equal(gs[k], osum[k]), f"summary {k} not bit-identical (rel err {e})"


def compare_tasks(traces, g, o_pt, osum, bitwise=True):
    """Per-task outputs of the traces whose status is OK."""
    ok = osum["status"] == 0
    mask = np.zeros(traces.n_tasks, bool)
    for t in np.nonzero(ok)[0]:
        mask[traces.offsets[t]:traces.offsets[t + 1]] = True
    nd_g, nd_o = g.node_defer[mask], o_pt["node_defer"][mask]
    bad = np.nonzero(nd_g != nd_o)[0]
    assert bad.size == 0, f"node_defer differs at {bad[:8]}: gpu {nd_g[bad[:8]]} oracle {nd_o[bad[:8]]}"
    assert np.array_equal(g.decision_idx[mask], o_pt["decision_idx"][mask]), "decision index differs"
    for k in ("completion", "start_f1"):
        gv, ov = getattr(g, k)[mask], o_pt[k][mask]
        e = rel_err(gv, ov)
        assert e <= REL_TOL, f"{k} rel err {e}"
        if bitwise:
            assert bits_equal(gv, ov), f"{k} not bit-identical (rel err {e})"


def run_both(N, S, traces, lp, fixed=None, outputs=True, cells=None, n_cells=1, eta_d=None):
    from paper_2507_21276_b200 import lemix
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, traces, lp, outputs=outputs, fixed_node=fixed, cells=cells, n_cells=n_cells,
                  eta_d=eta_d)
    osum, opt, ct, _ = oracle.run_batch(ef, eb, N, S, traces, oracle_params(lp), fixed_node=fixed, outputs=outputs,
                                        eta_d=eta_d)
    return g, osum, opt, ct


def check(N, S, traces, lp, fixed=None, outputs=True, bitwise=True, eta_d=None):
    g, osum, opt, ct = run_both(N, S, traces, lp, fixed, outputs, eta_d=eta_d)
    compare_summaries(g.summaries, osum, bitwise=bitwise)
    if outputs:
        compare_tasks(traces, g, opt, osum, bitwise=bitwise)
    return g, osum, ct
