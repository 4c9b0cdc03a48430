"""Algorithm 2 (ExecuteTaskMemoryAware; SURVEY.md §8f NEXT-1;
DESIGN.md reading R-mem) on the CUDA path through the C ABI, element by element
against the oracle: integers and indices bit-exact, fp64 times and summaries
bit-exact (north_star: within 1e-12 relative).  The worked examples of
SPEC.md:395-397 run through the CUDA path in tests/test_golden.py."""
from __future__ import annotations

import numpy as np
import pytest

import workload
from parity_util import check, compare_summaries, compare_tasks, run_both

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")

# Llama-8B stage: reference forward 0.055 s -> T_max = 10x, Delta_t = 0.1x
MEM = dict(mem_enable=1, mem_dt=0.0055, mem_tmax=0.55, mem_pen=8.8e-5)
POLICIES = [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE]


def P(**kw):
    return lemix.Params(**kw)


@pytest.mark.parametrize("cap", [300, 800, 2000])
@pytest.mark.parametrize("policy", POLICIES)
def test_sweep_shape_under_memory_pressure(cap, policy):
    parts = [workload.generate(workload.sweep_spec(rate), 6, seed_base=4000 + 6 * k)
             for k, rate in enumerate((40.0, 100.0, 160.0))]
    tr = workload.concat(parts)
    g, osum, _ = check(4, 2, tr, P(policy=policy, mem_cap=cap, **MEM))
    if cap <= 800:
        assert osum["n_mem_wait"].sum() > 0, "fixture should make tasks wait for memory"


@pytest.mark.parametrize("N,S", [(2, 4), (3, 3), (1, 2), (8, 1), (16, 8)])
def test_shapes_under_memory_pressure(N, S):
    tr = workload.generate(workload.tiny_spec(rate=60.0, n_inf=150), 3, seed_base=17)
    check(N, S, tr, P(mem_cap=500, **MEM))
    check(N, S, tr, P(policy=lemix.LMX_RR, mem_cap=500, **MEM))


def test_offload_regime():
    """T_max of one Delta_t and a cap below a single training micro-batch:
    every blocked forward is offloaded."""
    tr = workload.generate(workload.paper_spec(n_inf=2000, n_train=400), 2, seed_base=9)
    g, osum, _ = check(4, 2, tr, P(mem_cap=200, mem_dt=0.01, mem_tmax=0.01, mem_pen=1e-4, mem_enable=1))
    assert osum["n_offload"].sum() > 0


def test_unbounded_cap_equals_unlimited_memory():
    tr = workload.generate(workload.sweep_spec(150.0), 16, seed_base=23)
    ef, eb = workload.profile(4, 2)
    a = lemix.run(ef, eb, 4, 2, tr, P(), outputs=True)
    b = lemix.run(ef, eb, 4, 2, tr, P(mem_cap=1 << 40, **MEM), outputs=True)
    assert (b.summaries["n_mem_wait"] == 0).all()
    assert np.array_equal(a.node_defer, b.node_defer)
    assert a.completion.tobytes() == b.completion.tobytes()
    assert a.start_f1.tobytes() == b.start_f1.tobytes()


def test_mc_shape_with_memory_sampled():
    """2,048 MC-shaped traces (10k inference + 10k training) with the memory
    model on; 16 sampled traces against the oracle."""
    N, S = 4, 2
    tr = workload.mc_traces(2048, seed_base=77, with_out_len=False)
    lp = P(mem_cap=1024, **MEM)
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True)
    assert g.status == 0, g.error
    idx = np.array([0, 1, 500, 1023, 1024, 1500, 2046, 2047, 7, 99, 333, 777, 1111, 1666, 1999, 2000])
    sub = tr.subset(idx)
    import oracle
    from parity_util import oracle_params
    osum, opt, _, _ = oracle.run_batch(ef, eb, N, S, sub, oracle_params(lp))
    compare_summaries(g.summaries[idx], osum)

    class R:
        pass
    r = R()
    sel = np.concatenate([np.arange(tr.offsets[t], tr.offsets[t + 1]) for t in idx])
    r.node_defer, r.decision_idx = g.node_defer[sel], g.decision_idx[sel]
    r.completion, r.start_f1 = g.completion[sel], g.start_f1[sel]
    compare_tasks(sub, r, opt, osum)
    assert osum["n_mem_wait"].sum() > 0
