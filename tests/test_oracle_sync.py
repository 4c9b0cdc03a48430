"""Pin of the oracle's Separate checkpoint-synchronisation version model
(reading R-sync) by a recount
from the oracle's per-task outputs alone: for every inference task, the newest
checkpoint -- taken when the (k * interval)-th training task in release order
ends its backward, loaded sync_latency later -- among the training tasks
decided before it, that is loaded by its forward start.  The worked examples
of SPEC.md:422-423 are golden fixtures (tests/golden/spec42*_separate_sync*)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload


@pytest.mark.parametrize("interval,latency", [(1, 0.0), (3, 0.25), (10, 2.0)])
def test_separate_versions_recounted_from_outputs(interval, latency):
    tr = workload.generate(workload.sweep_spec(80.0, tasks=400), 4, seed_base=61)
    ef, eb = workload.profile(4, 2)
    par = oracle.OracleParams(policy=oracle.SEPARATE, sync_interval=interval, sync_latency=latency)
    for t in range(tr.n_traces):
        sub = tr.subset(np.array([t]))
        o = oracle.run_trace(ef, eb, 4, 2, sub.arrival, sub.lbk, sub.n_inf[0], par, want_paths=True)
        nI = int(sub.n_inf[0])
        dec = o["decision_idx"]
        train = np.arange(nI, len(dec))                     # release order = decision order (a chain)
        assert np.all(np.diff(dec[train]) > 0)
        ck_task = train[interval - 1::interval]            # the (k * interval)-th training tasks
        ck_avail = o["paths"][ck_task, 0, 3] + latency     # end_b^1 + latency
        total = 0
        for x in range(nI):
            sf = o["paths"][x, 0, 0]
            ks = [k + 1 for k in range(len(ck_task)) if dec[ck_task[k]] < dec[x] and ck_avail[k] <= sf]
            total += interval * (max(ks) if ks else 0)
        assert o["summary"]["sum_version"] == total


def test_sync_off_keeps_the_colocated_proxy():
    tr = workload.generate(workload.sweep_spec(80.0, tasks=300), 2, seed_base=5)
    ef, eb = workload.profile(4, 2)
    a = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=oracle.SEPARATE))[0]
    b = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=oracle.SEPARATE, sync_interval=0,
                                                                sync_latency=3.0))[0]
    assert a.tobytes() == b.tobytes()
    # co-located policies ignore the Separate sync model
    c = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams())[0]
    d = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(sync_interval=2, sync_latency=1.0))[0]
    assert c.tobytes() == d.tobytes()


def test_separate_dynamic_limits():
    """SeparateDynamic (R-sepdyn) with a threshold of 0 never
    switches to 1-3 (the static alpha partition); with a huge threshold it
    always runs 1-3: inference on node 0 only, training on the other nodes."""
    tr = workload.generate(workload.sweep_spec(100.0, tasks=300), 3, seed_base=17)
    ef, eb = workload.profile(4, 2)
    static = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=oracle.SEPARATE))
    never = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=oracle.SEPARATE, sep_dynamic=1,
                                                                     dyn_rate=0.0, dyn_window=5.0))
    assert np.array_equal(static[1]["node_defer"], never[1]["node_defer"])
    always = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(policy=oracle.SEPARATE, sep_dynamic=1,
                                                                      dyn_rate=1e30, dyn_window=5.0))
    node = always[1]["node_defer"] & 0xFFFF
    for t in range(tr.n_traces):
        a, b = tr.offsets[t], tr.offsets[t + 1]
        nI = tr.n_inf[t]
        assert set(node[a:a + nI]) == {0}
        assert set(node[a + nI:b]) == {1, 2, 3}
