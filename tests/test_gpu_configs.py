"""BASELINE.json configs at full size on the GPU, checked against the oracle on
sampled traces (the oracle computes them one by one) and through properties
that hold at any size.  Same C ABI and default launch configuration as
bench.py."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workload
from parity_util import compare_summaries, compare_tasks, oracle_params

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")


def _oracle_subset(N, S, tr, idx, lp):
    ef, eb = workload.profile(N, S)
    sub = tr.subset(idx)
    osum, opt, _, _ = oracle.run_batch(ef, eb, N, S, sub, oracle_params(lp))
    return sub, osum, opt


def _gpu_subset_tasks(g, tr, idx):
    """Per-task GPU outputs of the traces idx, in subset order."""
    class R:
        pass
    r = R()
    sel = np.concatenate([np.arange(tr.offsets[t], tr.offsets[t + 1]) for t in idx])
    r.node_defer = g.node_defer[sel]
    r.decision_idx = g.decision_idx[sel]
    r.completion = g.completion[sel]
    r.start_f1 = g.start_f1[sel]
    return r


def test_mc_full_size_sampled():
    """65,536 traces x 20k decisions (the bench workload), outputs on."""
    N, S = 4, 2
    tr = workload.mc_traces(65536, seed_base=1, with_out_len=False)
    lp = lemix.Params()
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True)
    assert g.status == 0
    assert (g.summaries["status"] == 0).all()
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.integers(0, 32768, 24), rng.integers(32768, 65536, 24), [0, 65535]]))
    sub, osum, opt = _oracle_subset(N, S, tr, idx, lp)
    compare_summaries(g.summaries[idx], osum)
    compare_tasks(sub, _gpu_subset_tasks(g, tr, idx), opt, osum)
    # properties over all traces: every task decided once, decision indices a permutation
    d = g.decision_idx.reshape(65536, 20000)
    assert (np.sort(d[:64], axis=1) == np.arange(20000)).all()
    assert (g.summaries["n_tasks"] == 20000).all()
    assert (g.summaries["slo_attainment"] >= 0).all() and (g.summaries["slo_attainment"] <= 1).all()


@pytest.mark.parametrize("policy", [lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE])
def test_sweep_full_size_sampled(policy):
    """4096 traces x 16 rates (1,000 tasks each), per-cell aggregates."""
    N, S = 4, 2
    parts = [workload.generate(workload.sweep_spec(rate), 4096, seed_base=1 + 4096 * k)
             for k, rate in enumerate(workload.SWEEP_RATES)]
    tr = workload.concat(parts)
    cells = np.repeat(np.arange(16, dtype=np.int32), 4096)
    lp = lemix.Params(policy=policy)
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True, cells=cells, n_cells=16)
    assert g.status == 0
    idx = np.array([c * 4096 + k for c in range(16) for k in (0, 4095)])
    sub, osum, opt = _oracle_subset(N, S, tr, idx, lp)
    compare_summaries(g.summaries[idx], osum)
    compare_tasks(sub, _gpu_subset_tasks(g, tr, idx), opt, osum)
    # the device cell reduction equals the host fold of the per-trace summaries
    from paper_2507_21276_b200 import dist as ldist
    host = ldist.cells_from_summaries(g.summaries, cells, 16)
    for k in lemix.CELL_INT:
        assert np.array_equal(g.cells[k], host[k]), k
    for k in lemix.CELL_F64:
        np.testing.assert_allclose(g.cells[k], host[k], rtol=1e-12, err_msg=k)


def test_paper_scale_ten_seeds_full():
    N, S = 4, 2
    tr = workload.generate(workload.paper_spec(), 10, seed_base=1)
    lp = lemix.Params()
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True)
    osum, opt, _, _ = oracle.run_batch(ef, eb, N, S, tr, oracle_params(lp))
    compare_summaries(g.summaries, osum)
    compare_tasks(tr, g, opt, osum)


def test_large_cluster_full_size_sampled():
    """64 nodes x 8 stages, 296 traces of 200k requests + 200k training."""
    N, S = 64, 8
    lp = lemix.Params(qcap=2048)
    parts = [workload.generate(workload.large_spec(rate=rate), 148, seed_base=7 + 148 * k)
             for k, rate in enumerate((1600.0, 3200.0))]
    tr = workload.concat(parts)
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True)
    print(f"large: {tr.n_tasks} decisions in {g.kernel_ms:.0f} ms kernel")
    idx = np.array([0, 148])
    sub, osum, opt = _oracle_subset(N, S, tr, idx, lp)
    compare_summaries(g.summaries[idx], osum)
    compare_tasks(sub, _gpu_subset_tasks(g, tr, idx), opt, osum)
    assert g.status == 0, g.error


def test_nccl_single_rank_allreduce_is_identity():
    """The NCCL path of lmx_allreduce_cells on a 1-rank communicator."""
    N, S = 4, 2
    tr = workload.generate(workload.tiny_spec(), 8, seed_base=3)
    ef, eb = workload.profile(N, S)
    ctx = lemix.Context(0)
    try:
        ctx.lmx_load_profile(N, S, ef, eb)
        ctx.lmx_load_traces(tr.offsets, tr.n_inf, tr.arrival, tr.lbk)
        ctx.lmx_set_params(lemix.Params())
        ctx.lmx_run()
        assert ctx.lmx_sync() == 0
        before = ctx.lmx_get_cells(1)
        comm = lemix.nccl_comm_init(1, lemix.nccl_unique_id(), 0, 0)
        ctx.lmx_allreduce_cells(comm)
        assert ctx.lmx_sync() == 0
        after = ctx.lmx_get_cells(1)
        lemix.nccl_comm_destroy(comm)
        assert before.tobytes() == after.tobytes()
    finally:
        ctx.close()


def test_rerun_reuses_streamed_inputs():
    """A second lmx_run on host-loaded traces reuses the copy (no re-stream)
    and gives identical results."""
    N, S = 4, 2
    tr = workload.generate(workload.sweep_spec(90.0), 64, seed_base=5)
    ef, eb = workload.profile(N, S)
    ctx = lemix.Context(0)
    try:
        ctx.lmx_load_profile(N, S, ef, eb)
        ctx.lmx_load_traces(tr.offsets, tr.n_inf, tr.arrival, tr.lbk)
        ctx.lmx_set_params(lemix.Params())
        ctx.lmx_run()
        assert ctx.lmx_sync() == 0
        a = ctx.lmx_get_summaries(tr.n_traces)
        ctx.lmx_run()
        assert ctx.lmx_sync() == 0
        b = ctx.lmx_get_summaries(tr.n_traces)
        assert a.tobytes() == b.tobytes()
    finally:
        ctx.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_runs_equal_single_run(world):
    """SURVEY.md §8(e) / §4 "fake backend": the P strided shards bench.py's
    ranks would own, run one after another on this GPU, reproduce the single
    run's per-trace outputs bit for bit, and their host-side sum of the
    per-cell blocks equals the single run's cells (integers exactly, fp64
    within 1e-12 relative) -- the result the one NCCL all-reduce returns."""
    from paper_2507_21276_b200 import dist as ldist
    N, S = 4, 2
    parts = [workload.generate(workload.sweep_spec(rate), 96, seed_base=500 + 96 * k)
             for k, rate in enumerate(workload.SWEEP_RATES)]
    tr = workload.concat(parts)
    cells = np.repeat(np.arange(16, dtype=np.int32), 96)
    lp = lemix.Params()
    ef, eb = workload.profile(N, S)
    whole = lemix.run(ef, eb, N, S, tr, lp, outputs=True, cells=cells, n_cells=16)
    assert whole.status == 0
    acc = None
    for rank in range(world):
        idx = ldist.strided_shard(tr.n_traces, rank, world)
        sub = tr.subset(idx)
        g = lemix.run(ef, eb, N, S, sub, lp, outputs=True, cells=cells[idx], n_cells=16)
        assert g.status == 0
        assert g.summaries.tobytes() == whole.summaries[idx].tobytes()
        sel = np.concatenate([np.arange(tr.offsets[t], tr.offsets[t + 1]) for t in idx])
        assert np.array_equal(g.node_defer, whole.node_defer[sel])
        assert np.array_equal(g.decision_idx, whole.decision_idx[sel])
        assert g.completion.tobytes() == whole.completion[sel].tobytes()
        assert g.start_f1.tobytes() == whole.start_f1[sel].tobytes()
        if acc is None:
            acc = {k: g.cells[k].copy() for k in lemix.CELL_INT + lemix.CELL_F64}
        else:
            for k in lemix.CELL_INT + lemix.CELL_F64:
                acc[k] = acc[k] + g.cells[k]
    for k in lemix.CELL_INT:
        assert np.array_equal(acc[k], whole.cells[k]), k
    for k in lemix.CELL_F64:
        np.testing.assert_allclose(acc[k], whole.cells[k], rtol=1e-12, err_msg=k)


def test_sweep_separate_sync_full_size_sampled():
    """The sweep config (4096 traces x 16 rates) under Separate with
    checkpoint synchronisation every 100 training tasks."""
    N, S = 4, 2
    parts = [workload.generate(workload.sweep_spec(rate), 4096, seed_base=1 + 4096 * k)
             for k, rate in enumerate(workload.SWEEP_RATES)]
    tr = workload.concat(parts)
    lp = lemix.Params(policy=lemix.LMX_SEPARATE, sync_interval=100, sync_latency=1.5)
    ef, eb = workload.profile(N, S)
    g = lemix.run(ef, eb, N, S, tr, lp, outputs=True)
    assert g.status == 0
    idx = np.array([c * 4096 + k for c in range(16) for k in (0, 4095)])
    sub, osum, opt = _oracle_subset(N, S, tr, idx, lp)
    compare_summaries(g.summaries[idx], osum)
    compare_tasks(sub, _gpu_subset_tasks(g, tr, idx), opt, osum)
    assert osum["sum_version"].sum() > 0


def test_parameter_sweep_cells():
    """NEXT-4 parameter study (Fig. 15, lambda1 / lambda2 / tau):
    one run with per-cell parameters equals, trace by trace, the oracle run
    with each cell's parameters."""
    N, S = 4, 2
    grid = [(l1, l2, tau) for l1 in (0.5, 1.0, 4.0) for l2 in (0.0, 1.0, 10.0) for tau in (-0.02, 0.0, 0.05)]
    K = len(grid)
    tr = workload.generate(workload.sweep_spec(120.0), 4 * K, seed_base=900)
    cells = np.repeat(np.arange(K, dtype=np.int32), 4)
    ef, eb = workload.profile(N, S)
    cp = {"lambda1": [g[0] for g in grid], "lambda2": [g[1] for g in grid], "tau": [g[2] for g in grid]}
    g = lemix.run(ef, eb, N, S, tr, lemix.Params(), outputs=True, cells=cells, n_cells=K, cell_params=cp)
    assert g.status == 0
    for k, (l1, l2, tau) in enumerate(grid):
        idx = np.nonzero(cells == k)[0]
        sub, osum, opt = _oracle_subset(N, S, tr, idx, lemix.Params(lambda1=l1, lambda2=l2, tau=tau))
        compare_summaries(g.summaries[idx], osum)
        compare_tasks(sub, _gpu_subset_tasks(g, tr, idx), opt, osum)
    # the cells differ (the parameters matter)
    assert len({g.summaries["n_slo_met"][cells == k].sum() for k in range(K)}) > 1
