"""Randomised parity sweep (seeded): random cluster shapes, policies, scheduler
parameters and model switches (Algorithm 2 memory, Separate sync / dynamic
partition, per-cell parameters), CUDA path vs oracle element by element."""
from __future__ import annotations

import numpy as np
import pytest

import workload
from parity_util import check

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")


def _case(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 24, 33]))
    S = int(rng.choice([1, 2, 3, 4, 6, 8]))
    pol = int(rng.choice([lemix.LMX_LEMIX, lemix.LMX_RR, lemix.LMX_SEPARATE] if N > 1 else [lemix.LMX_LEMIX,
                                                                                           lemix.LMX_RR]))
    kw = dict(policy=pol, lambda1=float(rng.choice([0.5, 1.0, 2.0])), lambda2=float(rng.choice([0.0, 1.0, 3.0])),
              tau=float(rng.choice([-0.01, 0.0, 0.02])), deprioritize=int(rng.integers(0, 2)),
              slo_mult=float(rng.choice([2.0, 5.0])), sigma_floor=float(rng.choice([1.0, 10.0])),
              lc0=float(rng.choice([0.0, 0.3989])), alpha=float(rng.choice([0.25, 0.5, 0.75])))
    if rng.random() < 0.35:
        kw.update(mem_enable=1, mem_cap=int(rng.choice([200, 600, 2000])), mem_dt=0.005,
                  mem_tmax=float(rng.choice([0.01, 0.05, 0.5])), mem_pen=float(rng.choice([0.0, 1e-4])))
    if pol == lemix.LMX_SEPARATE and rng.random() < 0.6:
        kw.update(sync_interval=int(rng.choice([1, 5, 50])), sync_latency=float(rng.choice([0.0, 0.5])))
    if pol == lemix.LMX_SEPARATE and rng.random() < 0.5:
        kw.update(sep_dynamic=1, dyn_rate=float(rng.choice([10.0, 50.0, 150.0])), dyn_window=2.0)
    rate = float(rng.choice([20.0, 60.0, 120.0, 200.0]))
    tasks = int(rng.choice([100, 300, 600]))
    tr = workload.generate(workload.sweep_spec(rate, alpha=float(rng.choice([0.2, 0.5, 0.8])), tasks=tasks),
                           int(rng.integers(1, 6)), seed_base=int(rng.integers(1, 10_000)))
    return N, S, tr, kw


@pytest.mark.parametrize("seed", range(96))
def test_random_configuration(seed):
    N, S, tr, kw = _case(seed)
    kw.setdefault("qcap", 4096)
    check(N, S, tr, lemix.Params(**kw))
