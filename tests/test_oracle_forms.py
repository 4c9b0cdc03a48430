"""The fp64 forms DESIGN.md R-stat (reciprocals: inv_c = 1/cnt, mu = sum*inv_c,
1/sigma, k = (0.5/sigma)/sigma, c = (1/sigma)/sqrt(2 pi)) and R-exp (Estrin
evaluation of the degree-13 Taylor polynomial) were adopted for speed after the
first kernel existed.  SURVEY.md 8c.4 states the textbook forms (mu = sum/cnt,
k = 0.5/(sigma^2), c = 1/(sigma sqrt(2 pi)), Horner).  Both are within a few
ulp of the exact Eq. 2; this test shows the choice changes
no scheduling result: an oracle built with -DORC_TEXTBOOK (same source, only
those two expressions swapped) makes the same decision on every task, with
the same times and the same summaries, over > 1 M decisions of the MC, sweep
and large-cluster workloads.  Only the LC values themselves (and so f) may
differ in the last bits."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload

INT = ("n_tasks", "n_slo_met", "n_deferrals", "active_nodes", "sum_version", "status")
F64 = ("makespan", "throughput", "sum_ttft", "mean_ttft", "slo_attainment", "mean_util", "mean_len_std")


def _same(N, S, tr, par):
    ef, eb = workload.profile(N, S)
    a = oracle.run_batch(ef, eb, N, S, tr, par)
    b = oracle.run_batch(ef, eb, N, S, tr, par, textbook=True)
    for k in ("node_defer", "decision_idx"):
        assert np.array_equal(a[1][k], b[1][k]), k
    for k in ("completion", "start_f1"):
        assert np.array_equal(a[1][k].view(np.int64), b[1][k].view(np.int64)), k
    for k in INT:
        assert np.array_equal(a[0][k], b[0][k]), k
    for k in F64:
        assert np.array_equal(a[0][k].view(np.int64), b[0][k].view(np.int64)), k
    assert a[2]["lc_exp"] > 0
    return tr.n_tasks


def test_exp_forms_agree_within_two_ulp():
    t = np.concatenate([np.linspace(0, 40, 20001), np.geomspace(1e-12, 700, 5001)])
    a = np.array([oracle.exp_neg(x) for x in t])
    b = np.array([oracle.exp_neg(x, textbook=True) for x in t])
    ulp = np.abs(a.view(np.int64) - b.view(np.int64))
    assert ulp.max() <= 2   # each is within 2 ulp of libm exp (test_oracle_units)


def test_textbook_forms_change_no_decision():
    n = 0
    # MC (the bench workload): 32 Poisson + 32 bursty traces x 20k decisions
    n += _same(4, 2, workload.concat([
        workload.generate(workload.mc_spec(False), 32, seed_base=1),
        workload.generate(workload.mc_spec(True), 32, seed_base=1 + 32768)]), oracle.OracleParams())
    # sweep: light to overloaded rates, under three (lambda1, lambda2, tau) settings
    sw = workload.concat([workload.generate(workload.sweep_spec(r), 16, seed_base=7 + int(r))
                          for r in workload.SWEEP_RATES])
    for kw in (dict(), dict(lambda1=0.25, lambda2=4.0), dict(lambda2=16.0, tau=0.005, lc0=0.3989422804014327)):
        n += _same(4, 2, sw, oracle.OracleParams(**kw))
    # large cluster shape: 64 x 8, heterogeneous lengths
    n += _same(64, 8, workload.generate(workload.large_spec(n_inf=6000), 2, seed_base=5), oracle.OracleParams())
    assert n >= 1_000_000
