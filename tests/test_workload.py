"""The shared input generator (workload/): determinism and distribution shape."""
from __future__ import annotations

import numpy as np

import workload


def test_deterministic_and_thread_independent():
    spec = workload.sweep_spec(50.0, tasks=500)
    a = workload.generate(spec, 64, seed_base=5, n_threads=1)
    b = workload.generate(spec, 64, seed_base=5, n_threads=7)
    assert np.array_equal(a.arrival.view(np.int64), b.arrival.view(np.int64))
    assert np.array_equal(a.lbk, b.lbk)
    c = workload.generate(spec, 64, seed_base=6, n_threads=4)
    assert not np.array_equal(a.arrival, c.arrival)
    # trace t of a batch == the same seed generated alone
    d = workload.generate(spec, 1, seed_base=5 + 17)
    t = a.trace(17)
    assert np.array_equal(t.arrival, d.arrival) and np.array_equal(t.lbk, d.lbk)


def test_layout_and_ranges():
    tr = workload.generate(workload.sweep_spec(80.0, tasks=1000), 8, seed_base=1)
    l, C, kind = workload.unpack(tr.lbk)
    assert l.min() >= 16 and l.max() <= 2048 and C.min() >= 1
    for t in range(tr.n_traces):
        o0, o1 = tr.offsets[t], tr.offsets[t + 1]
        nI = tr.n_inf[t]
        assert (kind[o0:o0 + nI] == 0).all() and (kind[o0 + nI:o1] == 1).all()
        assert np.all(np.diff(tr.arrival[o0:o0 + nI]) >= 0)


def test_poisson_mean_gap_spec45():
    # λ = 1, 1000 tasks -> mean inter-arrival within 1.0 ± 0.1
    spec = workload.WorkloadSpec(n_inf=1000, n_train=0, rate_inf=1.0)
    tr = workload.generate(spec, 20, seed_base=1)
    gaps = np.diff(tr.arrival.reshape(20, 1000), axis=1)
    assert abs(gaps.mean() - 1.0) < 0.1
    assert abs(gaps.std() / gaps.mean() - 1.0) < 0.1     # exponential: CV = 1


def test_bursty_cv():
    spec = workload.WorkloadSpec(n_inf=20000, n_train=0, rate_inf=50.0, bursty=True, cv=3.0)
    tr = workload.generate(spec, 4, seed_base=1)
    gaps = np.diff(tr.arrival.reshape(4, 20000), axis=1)
    assert abs(gaps.mean() * 50.0 - 1.0) < 0.15
    assert 2.4 < gaps.std() / gaps.mean() < 3.6


def test_training_fraction_spec69():
    # the training fraction tracks α (here fixed by construction)
    spec = workload.sweep_spec(100.0, alpha=0.3, tasks=10000)
    assert abs(spec.n_train / (spec.n_inf + spec.n_train) - 0.3) < 0.02


def test_lognormal_lengths_heavy_tail():
    spec = workload.WorkloadSpec(n_inf=50000, n_train=0, rate_inf=10.0)
    tr = workload.generate(spec, 1, seed_base=3)
    l = (tr.lbk & 0xFFF).astype(np.float64)
    assert 55 < np.median(l) < 75              # median 64
    assert np.mean(l) > np.median(l)           # right tail


def test_profile_table1():
    ef, eb = workload.profile(4, 2)
    assert ef[0] * 250000 == 0.11 and eb[0] * 250000 == 0.15    # PAPER.md:752, Llama-8B
    ef8, _ = workload.profile(64, 8)
    assert abs(ef8[0] * 8 - ef[0] * 2) < 1e-20


def test_mc_traces_half_bursty():
    tr = workload.mc_traces(8, seed_base=1, n_inf=2000, n_train=2000)
    assert tr.n_traces == 8 and tr.n_tasks == 8 * 4000
    g = [np.diff(tr.trace(t).arrival[:2000]) for t in range(8)]
    cv = [x.std() / x.mean() for x in g]
    assert max(cv[:4]) < 1.3 and min(cv[4:]) > 1.8


def test_mc_subset_equals_the_full_set_rows():
    """A rank's strided shard (bench.shard_traces, strong scaling) holds exactly
    the rows the full fixed seed set has for those trace indices."""
    full = workload.mc_traces(64, seed_base=7, n_inf=300, n_train=200, with_out_len=False)
    for rank, world in ((0, 1), (1, 4), (3, 4), (5, 8)):
        idx = np.arange(rank, 64, world)
        sub = workload.mc_traces_subset(idx, 64, 7, 300, 200, with_out_len=False)
        ref = full.subset(idx)
        assert np.array_equal(sub.offsets, ref.offsets)
        assert np.array_equal(sub.arrival.view(np.int64), ref.arrival.view(np.int64))
        assert np.array_equal(sub.lbk, ref.lbk)
        assert np.array_equal(sub.n_inf, ref.n_inf)
