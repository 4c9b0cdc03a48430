"""GPU (CUDA path through the C ABI) vs CPU oracle, element by element.

Integers and indices bit-exact; fp64 per-task times and summaries bit-exact by
construction and in any case within 1e-12 relative (north_star)."""
from __future__ import annotations

import numpy as np
import pytest

import workload
from parity_util import check, run_both, compare_summaries, compare_tasks

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")


def P(**kw):
    return lemix.Params(**kw)


POLICIES = [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE]


# ---------------------------------------------------------------- tiny config
@pytest.mark.parametrize("N,S", [(4, 2), (2, 4)])
@pytest.mark.parametrize("policy", POLICIES)
def test_tiny(N, S, policy):
    tr = workload.generate(workload.tiny_spec(), 1, seed_base=1)
    check(N, S, tr, P(policy=policy))


def test_tiny_fixed():
    tr = workload.generate(workload.tiny_spec(), 4, seed_base=11)
    rng = np.random.default_rng(5)
    fixed = rng.integers(0, 4, tr.n_tasks).astype(np.int32)
    check(4, 2, tr, P(policy=lemix.LMX_FIXED), fixed=fixed)


# ---------------------------------------------------------------- paper scale
def test_paper_scale():
    tr = workload.generate(workload.paper_spec(), 3, seed_base=1)
    check(4, 2, tr, P())


# ---------------------------------------------------------------- sweep
@pytest.mark.parametrize("policy", POLICIES)
def test_sweep_cells(policy):
    parts = [workload.generate(workload.sweep_spec(rate), 16, seed_base=1000 + 16 * k)
             for k, rate in enumerate(workload.SWEEP_RATES)]
    tr = workload.concat(parts)
    cells = np.repeat(np.arange(16, dtype=np.int32), 16)
    g, osum, opt, _ = run_both(4, 2, tr, P(policy=policy), cells=cells, n_cells=16)
    compare_summaries(g.summaries, osum)
    compare_tasks(tr, g, opt, osum)
    # per-cell integer aggregates equal the oracle's per-trace sums
    for c in range(16):
        sel = cells == c
        assert g.cells["n_slo_met"][c] == osum["n_slo_met"][sel].sum()
        assert g.cells["n_tasks"][c] == osum["n_tasks"][sel].sum()


# ---------------------------------------------------------------- variants
@pytest.mark.parametrize("N,S", [(1, 1), (1, 3), (3, 2), (5, 3), (8, 1), (16, 16), (33, 2), (100, 2)])
def test_shapes(N, S):
    tr = workload.generate(workload.tiny_spec(rate=40.0, n_inf=120), 3, seed_base=7)
    check(N, S, tr, P())
    if N >= 2:
        check(N, S, tr, P(policy=lemix.LMX_SEPARATE, alpha=0.3))
    check(N, S, tr, P(policy=lemix.LMX_RR))


@pytest.mark.parametrize("kw", [dict(deprioritize=0), dict(slo_mode=1, slo_const=0.05), dict(lc0=0.3989),
                                dict(tau=0.01), dict(tau=-0.02), dict(lambda1=2.0, lambda2=0.5),
                                dict(lambda2=0.0), dict(sigma_floor=25.0), dict(slo_mult=1.5)])
def test_params(kw):
    tr = workload.generate(workload.sweep_spec(120.0), 8, seed_base=21)
    check(4, 2, tr, P(**kw))


def test_edge_traces():
    tr = workload.from_lists([
        [],                                                  # empty
        [(0.0, 16, 1, 0)],                                   # one inference task
        [(0.0, 300, 2, 1)],                                  # one training task
        [(1.0, 64, 1, 0), (1.0, 64, 1, 0), (1.0, 64, 1, 0)],  # equal arrivals
        [(0.0, 100, 1, 1)] * 5,                              # training only, continuous
        [(0.5 * k, 2048, 255, k % 2) for k in range(40)],    # maximal w = 255 * 2048^2
        [(0.0, 1, 1, 0), (0.0, 1, 1, 1), (0.0, 1, 1, 0)],    # inference/training tie at t = 0
    ])
    for pol in POLICIES:
        check(4, 2, tr, P(policy=pol))
        check(1, 2, tr, P(policy=pol)) if pol != lemix.LMX_SEPARATE else None


def test_queue_capacity_overflow():
    tr = workload.generate(workload.sweep_spec(160.0), 8, seed_base=3)
    g, osum, _ = check(4, 2, tr, P(qcap=3))
    assert (osum["status"] == 6).any(), "fixture should overflow qcap=3"
    assert g.status == 6


def test_invalid_input_detected():
    tr = workload.generate(workload.tiny_spec(), 3, seed_base=2)
    tr.lbk[tr.offsets[1] + 5] = workload.pack(0, 1, 0)        # length 0 in trace 1
    g, osum, _ = check(4, 2, tr, P())
    assert osum["status"][1] == 1 and g.summaries["status"][1] == 1
    assert g.status == 1 and "trace 1" in g.error


# ---------------------------------------------------------------- large cluster
def test_large_cluster_trace():
    N, S = 64, 8
    tr = workload.generate(workload.large_spec(rate=1600.0, n_inf=20000), 2, seed_base=5)
    check(N, S, tr, P(qcap=1024))


# ---------------------------------------------------------------- Separate sync (NEXT-3)
@pytest.mark.parametrize("interval,latency", [(1, 0.0), (3, 0.25), (10, 2.0), (100, 1.5)])
def test_separate_checkpoint_sync(interval, latency):
    """Separate's checkpoint-synchronisation version model (
    DESIGN.md R-sync): sum_version bit-exact against the oracle."""
    parts = [workload.generate(workload.sweep_spec(rate), 8, seed_base=300 + 8 * k)
             for k, rate in enumerate((20.0, 80.0, 160.0))]
    tr = workload.concat(parts)
    g, osum, _ = check(4, 2, tr, P(policy=lemix.LMX_SEPARATE, sync_interval=interval, sync_latency=latency))
    assert (osum["sum_version"] > 0).any() or interval == 100


@pytest.mark.parametrize("rate,window", [(0.0, 5.0), (30.0, 2.0), (50.0, 10.0), (80.0, 1.0), (1e30, 3.0)])
def test_separate_dynamic(rate, window):
    """SeparateDynamic (DESIGN.md R-sepdyn) bit-exact against the
    oracle across rates that cross the threshold."""
    parts = [workload.generate(workload.sweep_spec(r), 6, seed_base=700 + 6 * k)
             for k, r in enumerate((20.0, 40.0, 60.0, 100.0, 160.0))]
    tr = workload.concat(parts)
    check(4, 2, tr, P(policy=lemix.LMX_SEPARATE, sep_dynamic=1, dyn_rate=rate, dyn_window=window))
    check(8, 2, tr, P(policy=lemix.LMX_SEPARATE, sep_dynamic=1, dyn_rate=rate, dyn_window=window,
                      sync_interval=7, sync_latency=0.5))


# ------------------------------------------- NEXT-2 / NEXT-4 / Eq. 4 reading
CB_POLICIES = [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE, lemix.LMX_MIXLUF]


@pytest.mark.parametrize("N,S", [(4, 2), (2, 4), (8, 8), (64, 2)])
@pytest.mark.parametrize("policy", CB_POLICIES)
def test_continuous_batching(N, S, policy):
    """Algorithm 3 batches + decode steps (DESIGN.md R-cb), bit-exact per
    request (node, decision, last-token time, start) and per trace (TTFT,
    SLO, TBT, batches)."""
    tr = workload.generate(workload.tiny_spec(rate=120.0, n_inf=300), 4, seed_base=17)
    lp = P(policy=policy, cb_cmax=8, cb_tw=workload.batch_timeout(S), luf_delay=0.002)
    g, osum, ct = check(N, S, tr, lp, eta_d=workload.decode_profile(N, S))
    assert osum["n_batches"].sum() < tr.n_inf.sum()     # some requests were batched
    assert osum["n_tbt"].sum() > 0


def test_continuous_batching_sweep_rates():
    tr = workload.concat([workload.generate(workload.sweep_spec(r), 3, seed_base=60 + int(r)) for r in (20.0, 160.0)])
    for policy in (lemix.LMX_LEMIX, lemix.LMX_SEPARATE):
        check(4, 2, tr, P(policy=policy, cb_cmax=16, cb_tw=0.05, sync_interval=5, sync_latency=0.3),
              eta_d=workload.decode_profile(4, 2))


@pytest.mark.parametrize("N,S", [(4, 2), (8, 8)])
def test_mix_luf(N, S):
    """Mix-LUF (R-luf) with and without the query latency."""
    tr = workload.generate(workload.tiny_spec(rate=60.0), 3, seed_base=23)
    for d in (0.0, 0.076):
        check(N, S, tr, P(policy=lemix.LMX_MIXLUF, luf_delay=d))


@pytest.mark.parametrize("N,S", [(4, 2), (2, 4), (8, 8)])
def test_eq4_mode1(N, S):
    """Eq. 4 reading R-14b (the training task's own forward counts)."""
    tr = workload.concat([workload.generate(workload.mc_spec(True, 400, 400, rate=150.0), 3, seed_base=31),
                          workload.generate(workload.tiny_spec(rate=80.0), 2, seed_base=32)])
    g, osum, ct = check(N, S, tr, P(eq4_mode=1))
    assert osum["n_deferrals"].sum() > 0


# ------------------------------------------- division / sqrt fast-path fallbacks
# The kernels form Eq. 3's quotient and Eq. 2's 1/cnt, sqrt and 1/sigma through
# branch-free replicas of ptxas's fast paths and recompute with the IEEE
# operations when a fast-path predicate fails (shortcut 5).
# A tiny tau makes IP = -tau on idle nodes, so Eq. 3's numerator is below the
# fast path's range in most decisions: the fallback branch runs, on the
# one-node-per-lane kernel (4 x 2), the wide kernel (40 x 8) and the generic
# tile kernel (Algorithm 2 on), with per-task outputs and summaries.
@pytest.mark.parametrize("kw", [dict(tau=2.0 ** -1000), dict(tau=2.0 ** -1000, lambda1=2.0 ** -60, lambda2=2.0 ** 40)])
@pytest.mark.parametrize("N,S,extra", [(4, 2, {}), (40, 8, {}),
                                       (4, 2, dict(mem_enable=1, mem_cap=800, mem_dt=0.0055, mem_tmax=0.55,
                                                   mem_pen=8.8e-5))])
def test_division_fallbacks(kw, N, S, extra):
    tr = workload.generate(workload.sweep_spec(120.0), 6, seed_base=41)
    check(N, S, tr, P(**kw, **extra))


# Summary-only runs take the LEAN instantiations: the same traces stop with the
# same status as the oracle and the same error (task index and field) as the
# per-task-output instantiations, on one-warp tiles and the wide kernel, for
# each kind of defect.
@pytest.mark.parametrize("N,S", [(4, 2), (40, 8)])
@pytest.mark.parametrize("defect", ["len0", "kind", "order", "negative"])
def test_invalid_input_summary_only(N, S, defect):
    tr = workload.generate(workload.tiny_spec(), 4, seed_base=3)
    o1, o2 = tr.offsets[1], tr.offsets[2]
    if defect == "len0":
        tr.lbk[o1 + 7] = workload.pack(0, 1, 0)
    elif defect == "kind":
        tr.lbk[o2 + 3] = workload.pack(64, 1, 1)                # an inference slot marked training
    elif defect == "order":
        tr.arrival[o1 + 9] = 0.5 * tr.arrival[o1 + 8]            # inference arrivals out of order
    else:
        tr.arrival[o2 + 2] = -1.0
    g, osum, _ = check(N, S, tr, P(), outputs=False)
    bad = np.nonzero(osum["status"] != 0)[0]
    assert len(bad) == 1
    assert np.array_equal(g.summaries["status"], osum["status"])
    g2, _, _ = check(N, S, tr, P(), outputs=True)                # the outputs path (validation first)
    assert g.error == g2.error and g.status == g2.status
