"""GPU stepwise parity (SURVEY.md §4 "GPU stepwise parity", §8(b) debug_level):
for every decision and every node, the kernel's Algorithm 1 II and R
 and Eq. 3 f must equal the oracle's
candidate table bit for bit -- not only the arg-best and the committed times.
Rows the algorithm does not evaluate (the baselines' other nodes, the
baselines' f) are NaN on both sides."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload
from parity_util import oracle_params

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")


def _stepwise(N, S, tr, lp, fixed=None, eta_d=None):
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True, fixed_node=fixed, eta_d=eta_d)
    assert g.cand is not None
    op = oracle_params(lp)
    n_checked = 0
    for t in range(tr.n_traces):
        a, b = tr.offsets[t], tr.offsets[t + 1]
        o = oracle.run_trace(ef, eb, N, S, tr.arrival[a:b], tr.lbk[a:b], tr.n_inf[t], op,
                             fixed_node=None if fixed is None else fixed[a:b], want_cand=True,
                             out_len=tr.out_len[a:b] if lp.cb_cmax > 0 else None, eta_d=eta_d)
        assert o["status"] == g.summaries["status"][t]
        oc, gc = o["cand"], g.cand[a:b]
        nan_o, nan_g = np.isnan(oc), np.isnan(gc)
        if o["status"] != 0:
            # decisions the trace reached agree; later rows are NaN on the GPU
            reached = ~np.all(nan_o, axis=(1, 2))
            oc, gc, nan_o, nan_g = oc[reached], gc[reached], nan_o[reached], nan_g[reached]
        bad = np.argwhere(nan_o != nan_g)
        assert bad.size == 0, f"trace {t}: evaluated candidates differ at (decision, node, field) {bad[:4]}"
        eq = oc.view(np.int64) == gc.view(np.int64)
        bad = np.argwhere(~eq & ~nan_o)
        assert bad.size == 0, (f"trace {t}: (II, R, f) differ at (decision, node, field) {bad[:4]}: "
                               f"gpu {gc[tuple(bad[0])]!r} oracle {oc[tuple(bad[0])]!r}")
        n_checked += int((~nan_o).sum())
    return n_checked


@pytest.mark.parametrize("N,S", [(4, 2), (2, 4), (1, 1), (8, 8), (64, 2)])
@pytest.mark.parametrize("policy", [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE])
def test_stepwise_tiny(N, S, policy):
    if policy == lemix.LMX_SEPARATE and N == 1:
        pytest.skip("Separate needs two nodes")
    tr = workload.generate(workload.tiny_spec(rate=60.0), 3, seed_base=21)
    assert _stepwise(N, S, tr, lemix.Params(policy=policy, debug_level=1)) > 0


def test_stepwise_paper_scale():
    """One paper-scale trace (20k bursty requests + 4k continuous C=4 micro-batches)."""
    tr = workload.generate(workload.paper_spec(), 1, seed_base=3)
    assert _stepwise(4, 2, tr, lemix.Params(debug_level=1)) > 4 * tr.n_tasks // 2


@pytest.mark.parametrize("policy", [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE])
def test_stepwise_sweep_sample(policy):
    """Sweep traces at a light and the heaviest rate, Eq. 4 and sync/dynamic Separate on."""
    tr = workload.concat([workload.generate(workload.sweep_spec(r), 4, seed_base=100 + int(r))
                          for r in (20.0, 160.0)])
    kw = dict(sync_interval=5, sync_latency=0.3, sep_dynamic=1) if policy == lemix.LMX_SEPARATE else {}
    _stepwise(4, 2, tr, lemix.Params(policy=policy, debug_level=1, **kw))


def test_stepwise_params_and_memory():
    tr = workload.generate(workload.tiny_spec(rate=80.0, n_inf=150), 3, seed_base=9)
    for kw in (dict(lambda1=0.5, lambda2=3.0, tau=0.01, lc0=0.3989422804014327),
               dict(slo_mode=1, slo_const=0.2),
               dict(mem_enable=1, mem_cap=300, mem_dt=0.0055, mem_tmax=0.055, mem_pen=1e-4)):
        _stepwise(4, 2, tr, lemix.Params(debug_level=1, **kw))


def test_stepwise_fixed():
    tr = workload.generate(workload.tiny_spec(), 2, seed_base=13)
    fixed = np.random.default_rng(1).integers(0, 4, tr.n_tasks).astype(np.int32)
    _stepwise(4, 2, tr, lemix.Params(policy=lemix.LMX_FIXED, debug_level=1), fixed=fixed)


def test_debug_off_rejects_get_candidates():
    ef, eb = workload.profile(4, 2)
    tr = workload.generate(workload.tiny_spec(), 1, seed_base=1)
    ctx = lemix.Context(0)
    try:
        ctx.lmx_load_profile(4, 2, ef, eb)
        ctx.lmx_load_traces(tr.offsets, tr.n_inf, tr.arrival, tr.lbk)
        ctx.lmx_set_params(lemix.Params())
        ctx.lmx_run()
        ctx.lmx_sync()
        with pytest.raises(lemix.LemixError):
            ctx.lmx_get_candidates(np.zeros((tr.n_tasks, 4, 3)))
        with pytest.raises(lemix.LemixError):
            ctx.lmx_set_params(lemix.Params(debug_level=2))
    finally:
        ctx.close()


def test_response_time_zero_is_invalid():
    """A forward too short to move the clock past the dispatch time (a = 1e10 s,
    ulp 1.9e-6 s, dF = 4.4e-7 s) gives R = 0 and an undefined Eq. 3
    (SPEC.md:286): the trace stops with LMX_EINVAL on both sides, and the
    other traces of the batch are unaffected."""
    N, S = 4, 2
    ef, eb = workload.profile(N, S)
    good = workload.generate(workload.tiny_spec(), 1, seed_base=1)
    bad = workload.from_lists([[(1e10, 1, 1, 0), (0.0, 1, 1, 1)]])
    tr = workload.concat([good, bad])
    g = lemix.run(ef, eb, N, S, tr, lemix.Params(), outputs=True)
    osum, _, _, _ = oracle.run_batch(ef, eb, N, S, tr, oracle.OracleParams())
    assert g.status == lemix.LMX_EINVAL
    assert list(g.summaries["status"]) == list(osum["status"]) == [0, lemix.LMX_EINVAL]
    assert "R <= 0" in g.error


def test_stepwise_batching_luf_eq4():
    tr = workload.generate(workload.tiny_spec(rate=120.0, n_inf=250), 3, seed_base=41)
    ed = workload.decode_profile(4, 2)
    for kw in (dict(cb_cmax=8, cb_tw=workload.batch_timeout(2)), dict(eq4_mode=1)):
        _stepwise(4, 2, tr, lemix.Params(debug_level=1, **kw), eta_d=ed if "cb_cmax" in kw else None)
    _stepwise(4, 2, tr, lemix.Params(policy=lemix.LMX_MIXLUF, luf_delay=0.01, debug_level=1))
