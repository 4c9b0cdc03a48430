"""Invariants of the oracle's schedules on randomized medium traces
(SURVEY.md §4)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload


def run(N, S, tr, **kw):
    ef, eb = workload.profile(N, S)
    return oracle.run_trace(ef, eb, N, S, tr.arrival, tr.lbk, tr.n_inf[0], oracle.OracleParams(**{"qcap": 4096, **kw}),
                            want_paths=True)


CASES = [(4, 2, 40.0), (4, 2, 150.0), (2, 4, 60.0), (3, 3, 90.0), (6, 1, 200.0)]


@pytest.mark.parametrize("N,S,rate", CASES)
@pytest.mark.parametrize("policy", [oracle.LEMIX, oracle.RR, oracle.SEPARATE])
def test_schedule_invariants(N, S, rate, policy):
    tr = workload.generate(workload.sweep_spec(rate, tasks=600), 1, seed_base=int(rate) + N)
    o = run(N, S, tr, policy=policy)
    assert o["status"] == 0
    nI = int(tr.n_inf[0])
    m = tr.n_tasks
    P = o["paths"]
    node = o["node"]
    # every task decided exactly once
    assert sorted(o["decision_idx"]) == list(range(m))
    # stage order and causality
    for t in range(m):
        assert P[t, 0, 0] >= tr.arrival[t]
        for s in range(S):
            assert P[t, s, 0] <= P[t, s, 1]
            if s + 1 < S:
                assert P[t, s, 1] <= P[t, s + 1, 0]
        if t >= nI:
            assert P[t, S - 1, 1] <= P[t, S - 1, 2]
            for s in range(S - 1):
                assert P[t, s + 1, 3] <= P[t, s, 2]
    # no two intervals overlap on any GPU (n, s)
    for n in range(N):
        for s in range(S):
            iv = [(P[t, s, 0], P[t, s, 1]) for t in range(m) if node[t] == n]
            iv += [(P[t, s, 2], P[t, s, 3]) for t in range(nI, m) if node[t] == n]
            iv.sort()
            for (a0, a1), (b0, b1) in zip(iv, iv[1:]):
                assert b0 >= a1, (n, s, (a0, a1), (b0, b1))
    # work conservation: busy time equals the sum of stage durations
    ef, eb = workload.profile(N, S)
    l = tr.lbk & 0xFFF
    C = (tr.lbk >> 12) & 0xFF
    w = (C.astype(np.int64) * l * l).astype(np.float64)
    busy = sum(ef[node[t] * S + s] * w[t] for t in range(m) for s in range(S))
    busy += sum(eb[node[t] * S + s] * w[t] for t in range(nI, m) for s in range(S))
    sm = o["summary"]
    assert abs(sm["mean_util"] * N * S * sm["makespan"] - busy) <= 1e-9 * busy
    assert 0 <= sm["active_nodes"] <= N
    assert 0.0 <= sm["slo_attainment"] <= 1.0 and 0.0 <= sm["mean_util"] <= 1.0


def test_determinism():
    tr = workload.generate(workload.paper_spec(n_inf=3000, n_train=800), 1, seed_base=3)
    a = run(4, 2, tr)
    b = run(4, 2, tr)
    for k in ("node_defer", "decision_idx", "completion", "start_f1", "paths"):
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8))
    assert a["summary"] == b["summary"]


def test_slo_attainment_monotone_in_slo_target():
    # on the same schedule, a smaller τ_R can only lower SLO attainment.
    # With Eq. 4 off the schedule does not depend on τ_R.
    tr = workload.generate(workload.sweep_spec(120.0, tasks=2000), 1, seed_base=4)
    prev = None
    for mult in (1.0, 2.0, 5.0, 20.0):
        o = run(4, 2, tr, slo_mult=mult, deprioritize=0)
        n = o["summary"]["n_slo_met"]
        if prev is not None:
            assert n >= prev
        prev = n


def test_inference_fcfs_preserved_by_deprioritisation():
    # Eq. 4 never reorders two inference tasks.
    total = 0
    for seed in range(1, 6):
        tr = workload.mc_traces(1, seed_base=seed, n_inf=4000, n_train=4000)
        o = run(4, 2, tr)
        total += o["summary"]["n_deferrals"]
        nI = int(tr.n_inf[0])
        assert np.all(np.diff(o["decision_idx"][:nI]) > 0)
        assert np.all(np.diff(o["decision_idx"][nI:]) > 0)
    assert total > 0


def test_lambda1_scaling_power_of_two_identical_choices_batch():
    tr = workload.generate(workload.sweep_spec(90.0, tasks=1000), 6, seed_base=12)
    ef, eb = workload.profile(4, 2)
    base = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(lambda1=1.0))
    for lam in (0.25, 4.0, 64.0):
        other = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(lambda1=lam))
        assert np.array_equal(base[1]["node_defer"], other[1]["node_defer"])
