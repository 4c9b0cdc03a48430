"""Pins of the oracle's continuous batching (Algorithm 3, PAPER.md:689-727;
DESIGN.md R-cb), Mix-LUF (R-luf) and the Eq. 4 reading R-14b beyond the
golden fixtures: reductions to the unbatched schedule and invariants of the
batch formation, checked on the workload generator's traces."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload

INT = ("n_tasks", "n_slo_met", "n_deferrals", "active_nodes", "sum_version", "status")
F64 = ("makespan", "throughput", "sum_ttft", "mean_ttft", "slo_attainment", "mean_util", "mean_len_std")


def _traces():
    return workload.concat([workload.generate(workload.sweep_spec(r, tasks=400), 3, seed_base=40 + int(r))
                            for r in (20.0, 80.0, 160.0)])


def _same(a, b):
    for k in ("node_defer", "decision_idx"):
        assert np.array_equal(a[1][k], b[1][k]), k
    for k in ("completion", "start_f1"):
        assert np.array_equal(a[1][k].view(np.int64), b[1][k].view(np.int64)), k
    for k in INT:
        assert np.array_equal(a[0][k], b[0][k]), k
    for k in F64:
        assert np.array_equal(a[0][k].view(np.int64), b[0][k].view(np.int64)), k


@pytest.mark.parametrize("policy", [oracle.LEMIX, oracle.RR, oracle.SEPARATE])
@pytest.mark.parametrize("cmax,tw", [(1, 0.3), (8, 0.0)])
def test_batches_of_one_without_decode_are_the_unbatched_schedule(policy, cmax, tw):
    """C = 1 (any T_w) or T_w = 0 (any C) makes every batch a single request
    executed at its arrival; with no decode steps the schedule is the
    unbatched one, double for double."""
    tr = _traces()
    tr.out_len[:] = 0
    ef, eb = workload.profile(4, 2)
    ed = ef * 0.01
    base = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=policy))
    cb = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=policy, cb_cmax=cmax, cb_tw=tw), eta_d=ed)
    _same(base, cb)
    assert (cb[0]["n_batches"] == tr.n_inf).all()
    assert (cb[0]["n_tbt"] == 0).all()


def test_batch_formation_invariants():
    """Members of a batch are consecutive requests sharing one decision and
    node, at most C of them, dispatched no earlier than their arrivals and no
    later than the batch's first arrival + T_w; a full batch's last member
    arrived no later than the first + T_w (Algorithm 3 lines 7-9)."""
    tr = workload.generate(workload.mc_spec(True, 3000, 3000, rate=120.0), 2, seed_base=5)
    ef, eb = workload.profile(4, 2)
    C, tw = 6, 0.05
    for t in range(tr.n_traces):
        a, b = tr.offsets[t], tr.offsets[t + 1]
        nI = tr.n_inf[t]
        o = oracle.run_trace(ef, eb, 4, 2, tr.arrival[a:b], tr.lbk[a:b], nI,
                             oracle.OracleParams(cb_cmax=C, cb_tw=tw), want_paths=True, out_len=tr.out_len[a:b],
                             eta_d=ef * 0.002)
        assert o["status"] == 0
        dec = o["decision_idx"][:nI]
        arr = tr.arrival[a:a + nI]
        start = o["paths"][:nI, 0, 0]
        sizes = []
        k = 0
        while k < nI:
            e = k
            while e + 1 < nI and dec[e + 1] == dec[k]:
                e += 1
            sizes.append(e - k + 1)
            assert e - k + 1 <= C
            assert len(set(o["node"][k:e + 1])) == 1
            assert np.all(arr[k:e + 1] < arr[k] + tw) or e == k
            # started (stage 1) no earlier than the last member's arrival
            assert start[k] >= arr[e]
            k = e + 1
        assert o["summary"]["n_batches"] == len(sizes)
        assert max(sizes) > 1                          # the bursty trace does batch
        # decode: a request's last token is at or after its first
        ttft_end = o["paths"][:nI, 1, 1]
        assert np.all(o["completion"][:nI] >= ttft_end)


def test_luf_zero_delay_picks_least_committed_node():
    """Mix-LUF with no query latency dispatches at the event time and always
    picks a node with the least busy time committed so far."""
    tr = workload.generate(workload.sweep_spec(80.0, tasks=300), 2, seed_base=3)
    ef, eb = workload.profile(4, 2)
    for t in range(tr.n_traces):
        a, b = tr.offsets[t], tr.offsets[t + 1]
        nI = tr.n_inf[t]
        o = oracle.run_trace(ef, eb, 4, 2, tr.arrival[a:b], tr.lbk[a:b], nI,
                             oracle.OracleParams(policy=oracle.MIXLUF), want_paths=True)
        assert o["status"] == 0
        order = np.argsort(o["decision_idx"])
        busy = np.zeros(4)
        w = (tr.lbk[a:b] & 0xFFF).astype(np.float64) ** 2 * ((tr.lbk[a:b] >> 12) & 0xFF)
        for task in order:
            n = o["node"][task]
            assert busy[n] == busy.min() and n == int(np.argmin(busy))
            busy[n] += ef[n * 2] * w[task] + ef[n * 2 + 1] * w[task]
            if task >= nI:
                busy[n] += eb[n * 2] * w[task] + eb[n * 2 + 1] * w[task]
        # dispatched at the event time: inference starts no earlier than arrival
        assert np.all(o["paths"][:nI, 0, 0] >= tr.arrival[a:a + nI])


def test_eq4_mode1_defers_at_least_as_often():
    """R-14b's inner term is never smaller than R-14's (it adds the training
    task's own forward), so it defers at least as often on the same traces."""
    tr = workload.generate(workload.mc_spec(True, 2000, 2000, rate=100.0), 2, seed_base=9)
    ef, eb = workload.profile(4, 2)
    d0 = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(eq4_mode=0))[0]["n_deferrals"].sum()
    d1 = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(eq4_mode=1))[0]["n_deferrals"].sum()
    assert d1 >= d0 and d1 > 0
