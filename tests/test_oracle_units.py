"""Pins of the CPU oracle against values the paper / SPEC.md fix by hand.

Every expected number below is either printed in SPEC.md / SURVEY.md §8c.7
(cited) or derived by hand in the comment next to it; none comes from the
oracle or the CUDA path.  Runs without a GPU.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workload
from workload import from_lists

INF = math.inf


def run1(N, S, eta_f, eta_b, trace, **kw):
    tr = from_lists([trace])
    par = oracle.OracleParams(**kw)
    ef = np.broadcast_to(np.asarray(eta_f, np.float64), (N * S,)).copy()
    eb = np.broadcast_to(np.asarray(eta_b, np.float64), (N * S,)).copy()
    o = oracle.run_trace(ef, eb, N, S, tr.arrival, tr.lbk, tr.n_inf[0], par, want_paths=True, want_cand=True)
    return tr, o


def ulp_diff(a, b):
    ia = np.float64(a).view(np.int64)
    ib = np.float64(b).view(np.int64)
    return abs(int(ia) - int(ib))


# ------------------------------------------------------------------ exp_neg [R-exp]
def test_exp_neg_exact_points():
    assert oracle.exp_neg(0.0) == 1.0
    assert oracle.exp_neg(700.5) == 0.0
    assert oracle.exp_neg(1e9) == 0.0


def test_exp_neg_within_2ulp_of_libm():
    rng = np.random.default_rng(0)
    ts = np.concatenate([rng.uniform(0, 1, 20000), rng.uniform(0, 50, 20000), rng.uniform(0, 700, 20000),
                         np.array([0.5, 1.0, 2.0, math.log(2), 10.0, 699.99])])
    worst = max(ulp_diff(oracle.exp_neg(t), math.exp(-t)) for t in ts)
    assert worst <= 2, worst


# ------------------------------------------------------------------ latency model
def test_single_task_ttft_is_sum_of_stage_forwards():
    # SPEC.md:467 [TRIVIAL]: one task, no contention -> TTFT = sum_s Δ_F, SLO 1.0
    # empty node, a = 0, S = 2, η_F = 1e-4, C = 1, ℓ = 100 -> II = 0, R = 2.0
    tr, o = run1(1, 2, 1e-4, 2e-4, [(0.0, 100, 1, 0)])
    assert o["cand"][0, 0, 0] == 0.0          # II
    assert o["cand"][0, 0, 1] == 2.0          # R
    assert o["completion"][0] == 2.0
    s = o["summary"]
    assert s["n_slo_met"] == 1 and s["slo_attainment"] == 1.0
    assert s["mean_ttft"] == 2.0


def test_predictor_table1_values():
    # η_F = 1.2e-7, η_B = 1.6e-7 at C = 1, ℓ = 500 -> 0.03 s / 0.04 s (GPT-400M, Table 1)
    tr, o = run1(1, 1, 1.2e-7, 1.6e-7, [(0.0, 500, 1, 1)], deprioritize=0)
    p = o["paths"][0, 0]
    assert p[0] == 0.0 and p[1] == 0.03          # forward [0, 0.03]
    assert p[2] == 0.03 and p[3] == 0.03 + 0.04  # backward right after it
    # doubling C doubles, doubling ℓ quadruples
    _, o2 = run1(1, 1, 1.2e-7, 1.6e-7, [(0.0, 500, 2, 0)])
    _, o4 = run1(1, 1, 1.2e-7, 1.6e-7, [(0.0, 1000, 1, 0)])
    assert o2["completion"][0] == 2 * 0.03 and o4["completion"][0] == 1.2e-7 * 1e6


# ------------------------------------------------------------------ Algorithm 1
def test_alg1_postpone_and_offset_spec202():
    # one stage, a training backward occupies [5, 7], prev.end_f = 5,
    # new forward of 1 -> postponed to [7, 8], II contribution (7-5) - 2 = 0.
    # Build: η_F = 1, η_B = 0.4; T1 (w = 5): forward [0, 5], backward [5, 7];
    # inference I (w = 1) arrives at 4.
    tr, o = run1(1, 1, 1.0, 0.4, [(4.0, 1, 1, 0), (0.0, 1, 5, 1)])
    # tasks reordered inference-first: index 0 = I, index 1 = T1
    assert list(o["paths"][1, 0]) == [0.0, 5.0, 5.0, 7.0]
    assert list(o["paths"][0, 0, :2]) == [7.0, 8.0]
    dec_I = o["decision_idx"][0]
    assert o["cand"][dec_I, 0, 0] == 0.0          # II
    assert o["cand"][dec_I, 0, 1] == 4.0          # R = 8 - 4


def _f1f2():
    # SURVEY.md §8c.7 fixture F1/F2 (hand-stepped): N = 1, S = 2, η_F = 1, η_B = 2, all w = 1,
    # T1 (a_min 0), I1 (a 0.5), T2 (a_min 0), I2 (a 7).
    return run1(1, 2, 1.0, 2.0, [(0.5, 1, 1, 0), (7.0, 1, 1, 0), (0.0, 1, 1, 1), (0.0, 1, 1, 1)])


def test_fixture_F1_F2_paths():
    tr, o = _f1f2()
    I1, I2, T1, T2 = 0, 1, 2, 3
    P = o["paths"]
    assert [list(P[T1, s]) for s in range(2)] == [[0, 1, 4, 6], [1, 2, 2, 4]]
    assert [list(P[I1, s, :2]) for s in range(2)] == [[1, 2], [4, 5]]
    assert [list(P[T2, s]) for s in range(2)] == [[2, 3, 8, 10], [5, 6, 6, 8]]
    assert [list(P[I2, s, :2]) for s in range(2)] == [[7, 8], [8, 9]]
    assert list(o["decision_idx"]) == [1, 3, 0, 2]
    cand = o["cand"][:, 0, :2]
    assert [tuple(c) for c in cand] == [(0, 2), (0, 4.5), (0, 5), (2, 2)]   # (II, R) per decision


def test_fixture_F1_F2_summary():
    tr, o = _f1f2()
    s = o["summary"]
    assert s["makespan"] == 10.0 and s["throughput"] == 0.4
    assert s["n_slo_met"] == 2 and s["mean_ttft"] == 3.25 and s["sum_ttft"] == 6.5
    assert s["mean_util"] == 0.8                    # busy 8 + 8 over 2 GPUs x 10 s
    assert s["sum_version"] == 1                    # I1 sees 0 finished backwards, I2 sees 1
    assert s["n_deferrals"] == 0 and s["active_nodes"] == 1


def test_fixture_F3_ii_quirk():
    # prev training forward [0,1],[1,2],
    # backward s2 [2,4], s1 [4,6]; new task w = 4 at a = 0.5 -> path [6,10],[10,14],
    # II = 3 + 8 = 11 (the consumed entry's stage-2 backward is not subtracted), R = 13.5.
    tr, o = run1(1, 2, 1.0, 2.0, [(0.5, 2, 1, 0), (0.0, 1, 1, 1)])
    assert [list(o["paths"][0, s, :2]) for s in range(2)] == [[6, 10], [10, 14]]
    d = o["decision_idx"][0]
    assert o["cand"][d, 0, 0] == 11.0 and o["cand"][d, 0, 1] == 13.5


def test_fit_before_pending_backward_is_inclusive():
    # [R-6] `end <= start_b` fits: a forward ending exactly at a pending backward's start
    # runs in the gap.  η_F = 1, η_B = 1, S = 1.  T1 (w = 2): forward [0,2], backward [2,4].
    # T2 (w = 3) released at 2: forward [4,7], backward [7,10].  I (w = 3) at 4: prev end 7 ->
    # scan: T1 consumed? forward [7,10] vs T1 sb 2 -> consumed (st = max(7,4) = 7);
    # T2 sb 7: en 10 <= 7 no -> consumed, st = 10 -> [10, 13].
    tr, o = run1(1, 1, 1.0, 1.0, [(4.0, 1, 3, 0), (0.0, 1, 2, 1), (0.0, 1, 3, 1)], deprioritize=0)
    assert list(o["paths"][0, 0, :2]) == [10.0, 13.0]
    # A task that fits exactly: inference w = 2 at t = 0.5 on a node whose T1 backward starts
    # at 2 (T1 forward [0,2]?) -> FIFO start 2 -> no gap.  Use two stages instead:
    # S = 2, η = 1: T1 (w=1) fwd [0,1],[1,2] bwd s2 [2,3] s1 [3,4];
    # I (w=1) at 1: stage 1 start max(1, 1) = 1, end 2 <= sb1 = 3 -> fits [1,2]; stage 2 [2,3]?
    # stage 2: start max(2, 2) = 2, end 3 <= sb2 = 2? no -> consumed -> start 3 -> [3, 4].
    tr, o = run1(1, 2, 1.0, 1.0, [(1.0, 1, 1, 0), (0.0, 1, 1, 1)])
    assert [list(o["paths"][0, s, :2]) for s in range(2)] == [[1, 2], [3, 4]]


# ------------------------------------------------------------------ Eq. 1 - 3
def test_eq1_branches_through_f():
    # F1/F2 decision of I2: II = 2, S = 2, a - a_[-1] = 7 - 1 = 6, R = 2, node history has
    # 3 tasks of length 1 -> sigma floored to 1 -> LC = 1/sqrt(2 pi).
    lc = 1.0 / math.sqrt(2.0 * math.pi)
    for tau, ip in [(0.0, -0.0), (1.0, -1.0), (-10.0, 5.0)]:   # IP = -max(1 - 6, tau)
        tr, o = run1(1, 2, 1.0, 2.0, [(0.5, 1, 1, 0), (7.0, 1, 1, 0), (0.0, 1, 1, 1), (0.0, 1, 1, 1)], tau=tau)
        f = o["cand"][3, 0, 2]
        assert abs(f - (ip + lc) / 2.0) <= 1e-15, (tau, f)


def test_eq2_gaussian_values_spec279():
    # σ = 10, ℓ = μ -> 0.03989...; μ = 100, σ = 10, ℓ = 110 -> 0.02420.
    # History lengths 90 and 110 give μ = 100 and population σ = 10.  Two nodes; node 0 takes
    # both history tasks (consolidation, f = LC0 = 0 ties -> lowest index), then probe tasks.
    # Far-apart arrivals: no interference, II = 0, IP = -max(0 - gap, 0) = 0, so f = LC / R.
    eta = 2.0 ** -20          # Δ_F = ℓ²·2^-20 and the arrival times are exact binary fractions
    for probe, expect in [(100, 0.039894228040143274), (110, 0.02419707245191434)]:
        trace = [(0.0, 90, 1, 0), (128.0, 110, 1, 0), (256.0, probe, 1, 0)]
        tr, o = run1(2, 1, eta, eta, trace)
        f, R = o["cand"][2, 0, 2], o["cand"][2, 0, 1]
        assert R == eta * probe * probe
        assert abs(f * R - expect) <= 4e-17, (probe, f * R)
        assert o["node"][2] == 0            # LC > 0 beats the fresh node's f = 0


def test_eq3_lambda_power_of_two_scaling_keeps_choices():
    # scaling λ1 by c > 0 keeps the argmax; with c = 2^k every f scales exactly.
    tr = workload.generate(workload.sweep_spec(120.0), 4, seed_base=9)
    ef, eb = workload.profile(4, 2)
    a = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(lambda1=1.0))
    b = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(lambda1=8.0))
    assert np.array_equal(a[1]["node_defer"], b[1]["node_defer"])
    assert np.array_equal(a[1]["completion"], b[1]["completion"])


def test_argbest_ties_lowest_index():
    # identical empty nodes -> node 0; every fresh node scores f = 0.
    tr, o = run1(3, 2, 1.0, 1.0, [(0.0, 10, 1, 0)])
    assert o["node"][0] == 0
    assert list(o["cand"][0, :, 2]) == [0.0, 0.0, 0.0]


# ------------------------------------------------------------------ Eq. 4
def test_eq4_defers_when_queues_end_late():
    # every node's queue ends at a'+10, forward needs 1, τ_R = 5 -> defer.
    # S = 1, η_F = η_B = 1.  I0 (w = 11) at 0: forward [0, 11].  T1 released at 0.5.
    # Next inference I1 at a' = 1 (w = 1): m = 11 + 1 = 12, 12 - 1 = 11 > τ_R = 5·1 -> defer.
    tr, o = run1(1, 1, 1.0, 1.0, [(0.0, 1, 11, 0), (1.0, 1, 1, 0), (0.5, 1, 1, 1)])
    assert o["defer"][2] == 1 and o["summary"]["n_deferrals"] == 1
    assert list(o["decision_idx"]) == [0, 1, 2]      # T1 placed after I1
    # SPEC.md:305 slack case: a' = 8 -> 12 - 8 = 4 <= 5 -> no deferral.
    tr, o = run1(1, 1, 1.0, 1.0, [(0.0, 1, 11, 0), (8.0, 1, 1, 0), (0.5, 1, 1, 1)])
    assert o["defer"][2] == 0 and list(o["decision_idx"]) == [0, 2, 1]
    # empty node anywhere -> -inf -> never defers
    tr, o = run1(2, 1, 1.0, 1.0, [(0.0, 1, 11, 0), (1.0, 1, 1, 0), (0.5, 1, 1, 1)])
    assert o["summary"]["n_deferrals"] == 0
    # the ablation flag turns it off ("w/o prioritize")
    tr, o = run1(1, 1, 1.0, 1.0, [(0.0, 1, 11, 0), (1.0, 1, 1, 0), (0.5, 1, 1, 1)], deprioritize=0)
    assert o["summary"]["n_deferrals"] == 0


# ------------------------------------------------------------------ baselines
def test_naivemix_rr_paper_example():
    # enqueue order 1', 1, 2, 2' -> NaiveMix puts {1', 2} on node 1 and {1, 2'} on node 2.
    # T1' at 0 (S1 forward [0, 1] releases T2' at 1); I1 at 0.5; I2 at 0.6.
    tr, o = run1(2, 2, 1.0, 1.0, [(0.5, 1, 1, 0), (0.6, 1, 1, 0), (0.0, 1, 1, 1), (0.0, 1, 1, 1)],
                 policy=oracle.RR)
    I1, I2, T1, T2 = 0, 1, 2, 3
    assert list(o["decision_idx"][[T1, I1, I2, T2]]) == [0, 1, 2, 3]
    assert o["node"][T1] == 0 and o["node"][I2] == 0 and o["node"][I1] == 1 and o["node"][T2] == 1
    # tasks 1..5 on N = 4 -> 0, 1, 2, 3, 0
    tr, o = run1(4, 1, 1.0, 1.0, [(float(k), 1, 1, 0) for k in range(5)], policy=oracle.RR)
    assert list(o["node"]) == [0, 1, 2, 3, 0]


@pytest.mark.parametrize("alpha,n_train_nodes", [(0.5, 2), (0.1, 1), (0.9, 3)])
def test_separate_partition_spec314(alpha, n_train_nodes):
    # N = 4, N_train = clamp(floor(4α + 0.5), 1, 3); inference nodes first
    trace = [(0.1 * k, 10, 1, 0) for k in range(12)] + [(0.0, 10, 1, 1) for _ in range(12)]
    tr, o = run1(4, 1, 1e-3, 1e-3, trace, policy=oracle.SEPARATE, alpha=alpha)
    n_inf_nodes = 4 - n_train_nodes
    inf_nodes = o["node"][:12]
    trn_nodes = o["node"][12:]
    assert set(inf_nodes) == set(range(n_inf_nodes))
    assert set(trn_nodes) == set(range(n_inf_nodes, 4))
    assert list(inf_nodes[:n_inf_nodes]) == list(range(n_inf_nodes))   # round-robin within the partition


def test_separate_needs_two_nodes():
    tr, o = run1(1, 1, 1.0, 1.0, [(0.0, 1, 1, 0), (0.0, 1, 1, 1)], policy=oracle.SEPARATE)
    assert o["status"] == oracle.EINVAL


# ------------------------------------------------------------------ backward planning, metrics
def test_backward_planning_spec210():
    # S = 1, end_f = 3, Δ_B = 0.5 -> backward [3, 3.5]
    tr, o = run1(1, 1, 3.0, 0.5, [(0.0, 1, 1, 1)])      # w = 1: Δ_F = 3, Δ_B = 0.5
    assert list(o["paths"][0, 0]) == [0.0, 3.0, 3.0, 3.5]
    # S = 2 symmetric -> end_b^1 = end_f^2 + 2 Δ_B
    tr, o = run1(1, 2, 3.0, 0.5, [(0.0, 1, 1, 1)])
    assert o["paths"][0, 1, 1] == 6.0 and o["completion"][0] == 6.0 + 2 * 0.5
    # two training tasks on one stage never overlap backwards
    tr, o = run1(1, 1, 1.0, 2.0, [(0.0, 1, 1, 1), (0.0, 1, 1, 1)])
    b1, b2 = o["paths"][0, 0, 2:], o["paths"][1, 0, 2:]
    assert b2[0] >= b1[1]


def test_metrics_zero_inference():
    # zero inference tasks -> SLO attainment 1.0
    tr, o = run1(1, 1, 1.0, 1.0, [(0.0, 1, 1, 1)])
    assert o["summary"]["slo_attainment"] == 1.0 and o["summary"]["mean_ttft"] == 0.0
    assert o["summary"]["makespan"] == 2.0 and o["summary"]["throughput"] == 0.5


def test_queue_capacity_overflow_is_reported():
    tr = workload.generate(workload.sweep_spec(160.0), 2, seed_base=3)
    ef, eb = workload.profile(4, 2)
    sums, _, _, st = oracle.run_batch(ef, eb, 4, 2, tr, oracle.OracleParams(qcap=2))
    assert st == oracle.EQCAP and (sums["status"] == oracle.EQCAP).all()
    assert (sums["n_slo_met"] == 0).all()       # a failed trace reports no metrics


def test_invalid_inputs_rejected():
    for bad in ([(0.0, 0, 1, 0)], [(0.0, 2049, 1, 0)], [(-1.0, 10, 1, 0)], [(math.nan, 10, 1, 0)],
                [(1.0, 10, 1, 0), (0.5, 10, 1, 0)]):
        tr, o = run1(1, 1, 1.0, 1.0, bad)
        assert o["status"] == oracle.EINVAL, bad


def test_response_time_zero_is_invalid_input():
    """Eq. 3 divides by R; R = 0 (a + dF rounds to a) is
    rejected as invalid input instead of scoring with inf/NaN."""
    ef, eb = workload.profile(4, 2)
    tr = workload.from_lists([[(1e10, 1, 1, 0), (0.0, 1, 1, 1)]])
    o = oracle.run_trace(ef, eb, 4, 2, tr.arrival, tr.lbk, tr.n_inf[0], oracle.OracleParams())
    assert o["status"] == 1   # ORC_EINVAL
    # one ulp more room and the same trace is fine: a = 1e9 (ulp 1.2e-7 < dF)
    tr = workload.from_lists([[(1e9, 1, 1, 0), (0.0, 1, 1, 1)]])
    o = oracle.run_trace(ef, eb, 4, 2, tr.arrival, tr.lbk, tr.n_inf[0], oracle.OracleParams())
    assert o["status"] == 0
