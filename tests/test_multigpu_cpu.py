"""World-size-2 gloo test of the multi-GPU host logic (sharding, the one
cross-rank summary reduction, max-over-ranks timing).  Runs on CPU; the
per-shard schedules come from the oracle standing in for each GPU.  The MC
case shards with bench.shard_traces -- the exact call bench.py makes on every
rank under torchrun (strong scaling: t = rank mod world of one fixed seed
set)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workload
from paper_2507_21276_b200 import dist as ldist

N, S = 4, 2
TRACES = 24


def _traces():
    parts = [workload.generate(workload.sweep_spec(rate, tasks=300), 4, seed_base=100 + 4 * k)
             for k, rate in enumerate((20.0, 60.0, 100.0, 140.0, 40.0, 160.0))]
    return workload.concat(parts)


def _cells_of(n):
    return np.arange(n) // 4   # 6 cells (rates) of 4 traces


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = _traces()
        idx = ldist.strided_shard(tr.n_traces, rank, world)
        sub = tr.subset(idx)
        ef, eb = workload.profile(N, S)
        sums, _, _, _ = oracle.run_batch(ef, eb, N, S, sub, oracle.OracleParams(), outputs=False)
        cells = ldist.cells_from_summaries(sums, _cells_of(tr.n_traces)[idx], n_cells=6)
        total = ldist.allreduce_cells(cells)
        slowest = ldist.max_over_ranks(float(rank + 1))
        q.put((rank, idx.tolist(), total, slowest))
    finally:
        dist.destroy_process_group()


def test_world2_sharding_and_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # the shards partition the traces
    all_idx = sorted(res[0][1] + res[1][1])
    assert all_idx == list(range(TRACES))
    assert not set(res[0][1]) & set(res[1][1])
    # both ranks hold the same reduced totals, equal to the single-process fold
    tr = _traces()
    ef, eb = workload.profile(N, S)
    sums, _, _, _ = oracle.run_batch(ef, eb, N, S, tr, oracle.OracleParams(), outputs=False)
    ref = ldist.cells_from_summaries(sums, _cells_of(TRACES), n_cells=6)
    for _, _, total, slowest in res:
        assert slowest == 2.0
        for k in ldist.CELL_INT:
            assert np.array_equal(total[k], ref[k]), k
        for k in ldist.CELL_F64:
            np.testing.assert_allclose(total[k], ref[k], rtol=1e-12, err_msg=k)


MC_TOTAL, MC_INF, MC_TRAIN = 16, 400, 300


def _mc_worker(rank, world, port, q):
    import sys

    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = bench.shard_traces(MC_TOTAL, rank, world, 3, MC_INF, MC_TRAIN, "strong")
        assert tr.n_traces == bench.traces_on_rank(MC_TOTAL, rank, world, "strong")
        ef, eb = workload.profile(N, S)
        sums, _, _, _ = oracle.run_batch(ef, eb, N, S, tr, oracle.OracleParams(), outputs=False)
        total = ldist.allreduce_cells(ldist.cells_from_summaries(sums))
        q.put((rank, total, sums["n_slo_met"].tolist()))
    finally:
        dist.destroy_process_group()


def test_world2_mc_strong_shards_equal_the_single_run():
    """The bench's strong-scaling shards of the fixed MC seed set, reduced
    across two ranks, give the single-process totals of the whole set."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = workload.mc_traces(MC_TOTAL, seed_base=3, n_inf=MC_INF, n_train=MC_TRAIN, with_out_len=False)
    ef, eb = workload.profile(N, S)
    sums, _, _, _ = oracle.run_batch(ef, eb, N, S, full, oracle.OracleParams(), outputs=False)
    ref = ldist.cells_from_summaries(sums)
    # per-trace results of each shard are the full run's rows t = rank mod 2
    for rank, _, slo in res:
        assert slo == sums["n_slo_met"][rank::world].tolist()
    for _, total, _ in res:
        for k in ldist.CELL_INT:
            assert np.array_equal(total[k], ref[k]), k
        for k in ldist.CELL_F64:
            np.testing.assert_allclose(total[k], ref[k], rtol=1e-12, err_msg=k)


def test_weak_seed_bases_disjoint():
    bases = [ldist.weak_seed_base(1, r, 65536) for r in range(8)]
    spans = [set(range(b, b + 65536)) for b in bases]
    for a in range(8):
        for b in range(a + 1, 8):
            assert not spans[a] & spans[b]


def test_strided_shard_rejects_bad_rank():
    with pytest.raises(ValueError):
        ldist.strided_shard(10, 2, 2)
