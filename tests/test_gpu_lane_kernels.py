"""The one-node-per-lane LeMix kernels (paper_2507_21276_b200/csrc/lemix_fast.cuh)
against the CPU oracle, element by element, over every shape class they take:
one-warp tiles (N <= 32, S in {1, 2, 4}) and the wide kernel (32 < N <= 128,
S in {2, 4, 8}, one trace per CTA of 2 or 4 warps).  The traces are chosen to
drive the paths these kernels add: deep training queues (entries past the
shared-memory window), stale prefixes set from the winning plan, CheckExecuted
over several entries, version counts, Eq. 4 deferrals under both readings
(R-14, R-14b), queue overflow and the stepwise candidate output (II, R, f of
every node at every decision)."""
from __future__ import annotations

import numpy as np
import pytest

import workload
from parity_util import check
from test_gpu_stepwise import _stepwise

pytestmark = pytest.mark.gpu

lemix = pytest.importorskip("paper_2507_21276_b200.lemix")

FAST = [(2, 1), (3, 4), (4, 1), (4, 4), (7, 2), (16, 4), (32, 1), (32, 2)]
WIDE = [(33, 4), (40, 8), (64, 4), (65, 2), (100, 8), (128, 8), (128, 2)]


def traces(seed, heavy=False):
    # heavy: continuous retraining (a_min = 0) at a high inference rate keeps
    # every node's Q_train deep (past the 4/8-entry windows)
    if heavy:
        spec = workload.WorkloadSpec(n_inf=400, n_train=400, rate_inf=400.0, bursty=True, cv=3.0,
                                     continuous_training=True)
    else:
        spec = workload.tiny_spec(rate=90.0, n_inf=250)
    return workload.generate(spec, 3, seed_base=seed)


def geometry(N, S, tr, lp):
    ctx = lemix.Context(0)
    try:
        ef, eb = workload.profile(N, S)
        lemix.run(ef, eb, N, S, tr, lp, ctx=ctx, outputs=False)
        return ctx.lmx_get_geometry()
    finally:
        ctx.close()


@pytest.mark.parametrize("N,S", FAST + WIDE)
def test_lane_kernels_bitexact(N, S):
    for heavy in (False, True):
        tr = traces(31 + N + S, heavy)
        check(N, S, tr, lemix.Params(qcap=4096))
        check(N, S, tr, lemix.Params(qcap=4096, eq4_mode=1, tau=-0.01))


@pytest.mark.parametrize("N,S", [(2, 1), (4, 2), (5, 4), (32, 2), (64, 8), (100, 2)])
def test_lane_kernels_summary_only(N, S):
    """Summary-only runs take the LEAN instantiation (no per-task outputs, no
    debug output, R-14, per-task tau_R compiled out): summaries bitwise."""
    for heavy in (False, True):
        check(N, S, traces(90 + N, heavy), lemix.Params(qcap=4096), outputs=False)


@pytest.mark.parametrize("N,S", [(4, 2), (32, 4), (64, 8), (128, 2)])
def test_lane_kernels_stepwise(N, S):
    """Every candidate's (II, R, f) at every decision, bitwise."""
    for heavy in (False, True):
        assert _stepwise(N, S, traces(77, heavy), lemix.Params(debug_level=1, qcap=4096)) > 0


def test_lane_kernels_queue_overflow():
    """A queue overflow (LMX_EQCAP) stops the trace at the same decision."""
    tr = traces(5, heavy=True)
    for N, S in ((4, 2), (64, 8)):
        g, osum, _ = check(N, S, tr, lemix.Params(qcap=2))
        assert (osum["status"] == 6).any()


@pytest.mark.parametrize("N,S,block", [(4, 2, 128), (32, 1, 128), (33, 4, 64), (64, 8, 64), (100, 8, 128)])
def test_lane_kernel_geometry(N, S, block):
    """Which kernel ran: one-warp tiles (128-thread CTAs, T = next_pow2(N)
    lanes per trace) or the wide kernel (one trace per CTA of 32 TW threads)."""
    grid, blk, lanes, smem = geometry(N, S, traces(3), lemix.Params())
    assert blk == block
