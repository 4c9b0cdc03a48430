"""Oracle vs the independent interval simulator, brute force over placements.

For random tiny traces (<= 8 tasks, N <= 4, S <= 3, mixed kinds, ties, random
coefficients) every forced placement (all N^k of them when small, a random
sample otherwise) is run through the oracle (policy FIXED) and through
tests/interval_sim.py; the planned forward and backward paths must agree
bitwise.  For LeMix (Eq. 4 off, so dispatch order follows the queue rule),
the response time R of every candidate node at every decision must equal the
simulator's one-step extension bitwise, and the chosen node must be the
arg-best of the oracle's own f with lowest-index ties.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle
from interval_sim import simulate_fixed
from workload import from_lists

ETAS = (0.5, 1.0, 1.5, 2.0, 3.0)


def random_instance(rng):
    N = int(rng.integers(1, 5))
    S = int(rng.integers(1, 4))
    k = int(rng.integers(1, 9))
    if rng.random() < 0.5:
        ef = rng.choice(ETAS, N * S)
        eb = rng.choice(ETAS, N * S)
    else:
        ef = rng.uniform(0.1, 3.0, N * S)
        eb = rng.uniform(0.1, 3.0, N * S)
    tasks = []
    for _ in range(k):
        kind = int(rng.random() < 0.5)
        a = float(rng.choice([0.0, 0.5, 1.0, 2.0, 3.5])) if rng.random() < 0.5 else float(rng.uniform(0, 6))
        tasks.append((a, int(rng.integers(1, 4)), int(rng.integers(1, 3)), kind))
    inf = sorted([t for t in tasks if t[3] == 0], key=lambda t: t[0])
    trn = [t for t in tasks if t[3] == 1]
    return N, S, ef, eb, inf + trn


def oracle_paths(N, S, ef, eb, tr, params, fixed=None):
    o = oracle.run_trace(ef, eb, N, S, tr.arrival, tr.lbk, tr.n_inf[0], params, fixed_node=fixed,
                         want_paths=True, want_cand=True)
    assert o["status"] == 0
    return o


def assert_paths_equal(o, paths, backs, n_inf, S):
    for task, p in paths.items():
        for s in range(S):
            assert o["paths"][task, s, 0] == p[s][0] and o["paths"][task, s, 1] == p[s][1], (task, s)
            if task >= n_inf:
                assert o["paths"][task, s, 2] == backs[task][s][0], (task, s, "sb")
                assert o["paths"][task, s, 3] == backs[task][s][1], (task, s, "eb")


def test_forced_placements_match_interval_simulator():
    rng = np.random.default_rng(2024)
    n_cases = 0
    for _ in range(160):
        N, S, ef, eb, tasks = random_instance(rng)
        tr = from_lists([tasks])
        k = len(tasks)
        if N ** k <= 256:
            placements = [np.array(p, np.int32) for p in itertools.product(range(N), repeat=k)]
        else:
            placements = [rng.integers(0, N, k).astype(np.int32) for _ in range(48)]
        for pl in placements:
            o = oracle_paths(N, S, ef, eb, tr, oracle.OracleParams(policy=oracle.FIXED), fixed=pl)
            paths, backs, _ = simulate_fixed(N, S, ef, eb, tr.arrival, tr.lbk, int(tr.n_inf[0]), pl)
            assert_paths_equal(o, paths, backs, int(tr.n_inf[0]), S)
            n_cases += 1
    assert n_cases > 5000


@pytest.mark.parametrize("seed", range(4))
def test_lemix_candidates_match_one_step_extensions(seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(150):
        N, S, ef, eb, tasks = random_instance(rng)
        tr = from_lists([tasks])
        for tau, lc0 in ((0.0, 0.0), (0.3, 0.2)):
            par = oracle.OracleParams(policy=oracle.LEMIX, deprioritize=0, tau=tau, lc0=lc0)
            o = oracle_paths(N, S, ef, eb, tr, par)
            placement = o["node"]
            paths, backs, probes = simulate_fixed(N, S, ef, eb, tr.arrival, tr.lbk, int(tr.n_inf[0]), placement,
                                                  probe_all=True)
            assert_paths_equal(o, paths, backs, int(tr.n_inf[0]), S)
            for task, Rs in probes.items():
                d = o["decision_idx"][task]
                cand = o["cand"][d]
                for n in range(N):
                    assert cand[n, 1] == Rs[n], (task, n, cand[n, 1], Rs[n])
                f = cand[:, 2]
                best = 0
                for n in range(1, N):
                    if f[n] > f[best]:
                        best = n
                assert placement[task] == best


def test_rr_and_separate_follow_their_rotation():
    rng = np.random.default_rng(7)
    for _ in range(100):
        N, S, ef, eb, tasks = random_instance(rng)
        tr = from_lists([tasks])
        o = oracle_paths(N, S, ef, eb, tr, oracle.OracleParams(policy=oracle.RR))
        order = np.argsort(o["decision_idx"])
        assert list(o["node"][order]) == [d % N for d in range(len(tasks))]
        paths, backs, _ = simulate_fixed(N, S, ef, eb, tr.arrival, tr.lbk, int(tr.n_inf[0]), o["node"])
        assert_paths_equal(o, paths, backs, int(tr.n_inf[0]), S)
