"""Pins of the oracle's Algorithm 2 (ExecuteTaskMemoryAware, PAPER.md:608-641;
DESIGN.md reading R-mem) that do not go through its own
code: the worked examples live in tests/golden/spec39{5,6,7}_*.json; here

* a cap that never binds reproduces the unlimited-memory schedule bit for bit
  ("demand below threshold -> Executed immediately");
* an interval-based recount of the memory held on every GPU at every executed
  forward start (activations of training tasks live on GPU (n, s) from their
  stage-s forward start to their stage-s backward end) never
  exceeds the cap for a forward that was not offloaded -- the admission rule
  of Algorithm 2 line 7, checked from the executed paths alone;
* executed intervals never overlap on a GPU, every stage follows the previous
  one, and a waited forward starts no earlier than Algorithm 1 planned it.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload
from workload import from_lists

MEM = dict(mem_enable=1, mem_dt=0.005, mem_tmax=0.05, mem_pen=2e-7)


def _run(N, S, tr, **kw):
    ef, eb = workload.profile(N, S)
    par = oracle.OracleParams(**kw)
    outs = []
    for t in range(tr.n_traces):
        sub = tr.subset(np.array([t]))
        outs.append(oracle.run_trace(ef, eb, N, S, sub.arrival, sub.lbk, sub.n_inf[0], par, want_paths=True))
    return outs, ef, eb


@pytest.mark.parametrize("policy", [oracle.LEMIX, oracle.RR])
def test_unbounded_cap_is_the_hot_path_schedule(policy):
    tr = workload.generate(workload.sweep_spec(140.0), 4, seed_base=31)
    free, _, _ = _run(4, 2, tr, policy=policy)
    big, _, _ = _run(4, 2, tr, policy=policy, mem_cap=1 << 40, **MEM)
    for a, b in zip(free, big):
        assert b["summary"]["n_mem_wait"] == 0 and b["summary"]["n_offload"] == 0
        assert np.array_equal(a["node_defer"], b["node_defer"])
        assert a["paths"].tobytes() == b["paths"].tobytes()
        assert a["completion"].tobytes() == b["completion"].tobytes()


@pytest.mark.parametrize("cap", [600, 1500, 4000])
@pytest.mark.parametrize("N,S", [(4, 2), (2, 3)])
def test_admissions_respect_the_cap(cap, N, S):
    tr = workload.generate(workload.sweep_spec(160.0, tasks=400), 3, seed_base=7 + cap)
    outs, ef, eb = _run(N, S, tr, mem_cap=cap, **MEM)
    waited = 0
    for t, o in enumerate(outs):
        assert o["status"] == 0
        sub = tr.subset(np.array([t]))
        nI = int(sub.n_inf[0])
        lbk = sub.lbk
        tok = ((lbk >> 12) & 0xFF).astype(np.int64) * (lbk & 0xFFF).astype(np.int64)
        w = tok * (lbk & 0xFFF).astype(np.int64)
        node = o["node"]
        P = o["paths"]
        waited += o["summary"]["n_mem_wait"]
        m = len(lbk)
        for n in range(N):
            on = np.nonzero(node == n)[0]
            for s in range(S):
                dF = ef[n * S + s] * w.astype(np.float64)
                dur = P[:, s, 1] - P[:, s, 0]
                off = dur != dF          # an offloaded forward carries the penalty (mem_pen > 0)
                # the memory held on GPU (n, s) when each forward starts
                for x in on:
                    t0 = P[x, s, 0]
                    held = 0
                    for q in on:
                        if q >= nI and q != x and not off[q] and P[q, s, 0] <= t0 < P[q, s, 3]:
                            held += tok[q]
                    if not off[x]:
                        assert held + tok[x] <= cap, (t, n, s, x, held, tok[x])
                # executed forwards and backwards never overlap on the GPU
                iv = [(P[x, s, 0], P[x, s, 1]) for x in on]
                iv += [(P[x, s, 2], P[x, s, 3]) for x in on if x >= nI]
                iv.sort()
                for (a0, a1), (b0, b1) in zip(iv, iv[1:]):
                    assert a1 <= b0, (t, n, s, (a0, a1), (b0, b1))
            for x in on:   # stage order
                for s in range(1, S):
                    assert P[x, s, 0] >= P[x, s - 1, 1]
        assert m == o["summary"]["n_tasks"]
    assert waited > 0, "the fixture should exercise memory waits"


def test_waits_never_start_earlier_than_planned():
    """A forward's executed start is >= the start Algorithm 1 planned for it
    (the candidate table of the chosen node records the planned R)."""
    tr = workload.generate(workload.sweep_spec(160.0, tasks=300), 2, seed_base=3)
    ef, eb = workload.profile(4, 2)
    par = oracle.OracleParams(mem_cap=1500, **MEM)
    for t in range(tr.n_traces):
        sub = tr.subset(np.array([t]))
        o = oracle.run_trace(ef, eb, 4, 2, sub.arrival, sub.lbk, sub.n_inf[0], par, want_paths=True, want_cand=True)
        nI = int(sub.n_inf[0])
        for x in range(nI):   # inference: R = end_f^S - a, planned vs executed
            d, n = o["decision_idx"][x], o["node"][x]
            planned_R = o["cand"][d, n, 1]
            executed_R = o["paths"][x, 1, 1] - sub.arrival[x]
            assert executed_R >= planned_R


def test_memory_params_validated():
    tr = from_lists([[(0.0, 10, 1, 0)]])
    ef, eb = workload.profile(1, 1)
    for bad in (dict(mem_dt=0.0), dict(mem_tmax=float("inf")), dict(mem_cap=-1), dict(mem_pen=-1.0),
                dict(mem_dt=1e-9, mem_tmax=1.0)):
        kw = dict(mem_enable=1, mem_cap=10, mem_dt=0.1, mem_tmax=1.0, mem_pen=0.0) | bad
        o = oracle.run_trace(ef, eb, 1, 1, tr.arrival, tr.lbk, tr.n_inf[0], oracle.OracleParams(**kw))
        assert o["status"] == oracle.EINVAL, bad


def test_without_algorithm2_the_cap_is_exceeded():
    """SPEC.md:550 (acceptance 6, the PAPER.md:1081 "w/o memory" ablation): on
    a saturating workload, unlimited admission checked post hoc against the
    cap has violating admissions, while Algorithm 2 has none
    (test_admissions_respect_the_cap)."""
    cap = 600
    tr = workload.generate(workload.sweep_spec(160.0, tasks=400), 2, seed_base=7 + cap)
    outs, ef, eb = _run(4, 2, tr)                      # memory model off
    violations = 0
    for t, o in enumerate(outs):
        sub = tr.subset(np.array([t]))
        nI = int(sub.n_inf[0])
        lbk = sub.lbk
        tok = ((lbk >> 12) & 0xFF).astype(np.int64) * (lbk & 0xFFF).astype(np.int64)
        P = o["paths"]
        for n in range(4):
            on = np.nonzero(o["node"] == n)[0]
            for s in range(2):
                for x in on:
                    t0 = P[x, s, 0]
                    held = sum(tok[q] for q in on if q >= nI and q != x and P[q, s, 0] <= t0 < P[q, s, 3])
                    violations += held + tok[x] > cap
    assert violations > 0
