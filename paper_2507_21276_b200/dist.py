"""Multi-GPU plumbing for the placement step.

Traces are independent units: they share no state and exchange nothing, so
ranks shard them and the only cross-rank exchange is one sum of the per-cell
summary aggregates at the end (done on device by lmx_allreduce_cells over
NCCL; `allreduce_cells` below is the torch.distributed equivalent used when
the library's communicator is not in play, e.g. the gloo CPU tests).

Two sharding modes:
  * weak  -- every rank owns its own `per_rank` seeded traces
             (seed_base + rank * per_rank + t); the bench's mode;
  * strong -- a fixed set of `n_traces` traces, rank r takes t = r mod world
             (interleaved, so every rank gets the same mix of rates/policies).
"""
from __future__ import annotations

import numpy as np

from .lemix import CELL_DTYPE, CELL_F64, CELL_INT


def weak_seed_base(seed_base: int, rank: int, per_rank: int) -> int:
    """First seed of rank `rank` when each rank owns `per_rank` traces."""
    return seed_base + rank * per_rank


def strided_shard(n_traces: int, rank: int, world: int) -> np.ndarray:
    """Trace indices owned by `rank` in strong-scaling mode (t = rank mod world)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return np.arange(rank, n_traces, world, dtype=np.int64)


def cells_to_blocks(cells: np.ndarray):
    """Split lmx_cell_summary records into the int64 and fp64 blocks that are
    all-reduced (the same layout lmx_allreduce_cells reduces on device)."""
    ib = np.stack([cells[k] for k in CELL_INT], axis=1).astype(np.int64)
    fb = np.stack([cells[k] for k in CELL_F64], axis=1).astype(np.float64)
    return ib, fb


def blocks_to_cells(ib: np.ndarray, fb: np.ndarray) -> np.ndarray:
    out = np.zeros(ib.shape[0], CELL_DTYPE)
    for j, k in enumerate(CELL_INT):
        out[k] = ib[:, j]
    for j, k in enumerate(CELL_F64):
        out[k] = fb[:, j]
    return out


def allreduce_cells(cells: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum cell aggregates over all ranks with torch.distributed (any backend)."""
    import torch
    import torch.distributed as dist

    ib, fb = cells_to_blocks(cells)
    ti = torch.from_numpy(ib)
    tf = torch.from_numpy(fb)
    if device is not None:
        ti, tf = ti.to(device), tf.to(device)
    dist.all_reduce(ti, group=group)
    dist.all_reduce(tf, group=group)
    return blocks_to_cells(ti.cpu().numpy(), tf.cpu().numpy())


def max_over_ranks(value: float, group=None, device=None) -> float:
    """The job's step time is the slowest rank's (timing rule)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def cells_from_summaries(summaries: np.ndarray, cell_of=None, n_cells: int = 1) -> np.ndarray:
    """Host-side cell aggregation with the same rules as the device reduction
    (sum over a cell's LMX_OK traces; failed traces only counted)."""
    out = np.zeros(n_cells, CELL_DTYPE)
    cell_of = np.zeros(len(summaries), np.int64) if cell_of is None else np.asarray(cell_of)
    for c in range(n_cells):
        s = summaries[cell_of == c]
        ok = s[s["status"] == 0]
        out["n_traces"][c] = len(s)
        out["n_failed"][c] = len(s) - len(ok)
        for k_out, k_in in (("n_tasks", "n_tasks"), ("n_inf", "n_inf"), ("n_train", "n_train"),
                            ("n_slo_met", "n_slo_met"), ("n_deferrals", "n_deferrals"),
                            ("sum_active_nodes", "active_nodes"), ("sum_version", "sum_version")):
            out[k_out][c] = ok[k_in].sum()
        for k_out, k_in in (("sum_makespan", "makespan"), ("sum_throughput", "throughput"),
                            ("sum_ttft", "sum_ttft"), ("sum_mean_ttft", "mean_ttft"),
                            ("sum_slo_attainment", "slo_attainment"), ("sum_mean_util", "mean_util"),
                            ("sum_mean_len_std", "mean_len_std")):
            acc = 0.0
            for v in ok[k_in]:
                acc = acc + float(v)
            out[k_out][c] = acc
    return out
