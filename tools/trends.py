"""Report-only trend checks of the scheduler (acceptance 2-5;
the paper's directional claims PAPER.md:569-573, 914, 921-926, 1075).

Runs the CPU oracle (test infrastructure) on seeded synthetic traces of the
sweep shape (N=4, S=2, Llama-8B profile, 1,000 tasks per trace, 10 seeds per
point) and writes the measured trends as JSON.  Nothing here is asserted and
nothing is tuned to pass ("do not tune the oracle to pass").

    python tools/trends.py [--out profiles/trends_r01.json] [--seeds 10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workload  # noqa: E402

N, S = 4, 2
POL = {"lemix": oracle.LEMIX, "rr": oracle.RR, "separate": oracle.SEPARATE}


def run(rate, alpha, seeds, **kw):
    tr = workload.generate(workload.sweep_spec(rate, alpha=alpha), seeds, seed_base=9000)
    ef, eb = workload.profile(N, S)
    sums, _, _, st = oracle.run_batch(ef, eb, N, S, tr, oracle.OracleParams(alpha=alpha, **kw), outputs=False)
    ok = sums["status"] == 0
    return {k: float(np.mean(sums[k][ok])) for k in ("throughput", "slo_attainment", "active_nodes", "mean_ttft",
                                                      "mean_util")} | {"failed": int((~ok).sum())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "trends_r01.json"))
    ap.add_argument("--seeds", type=int, default=10)
    a = ap.parse_args()
    k = a.seeds
    rep = {"workload": f"sweep shape: N={N}, S={S}, Llama-8B profile, 1,000 tasks/trace, {k} seeds per point, oracle",
           "note": "report-only (SPEC.md:546-549); rates are total task rates (tasks/s) of the Llama-8B profile"}
    # 2. throughput ordering at overload
    thr = {p: run(100.0, 0.5, k, policy=v)["throughput"] for p, v in POL.items()}
    rep["throughput_at_100"] = thr | {"lemix_ge_rr_ge_separate": thr["lemix"] >= thr["rr"] >= thr["separate"],
                                      "lemix_over_separate": thr["lemix"] / thr["separate"]}
    # 3. SLO attainment non-increasing in the rate
    slo = {p: [run(r, 0.5, k, policy=v)["slo_attainment"] for r in (10.0, 50.0, 100.0, 150.0)] for p, v in POL.items()}
    rep["slo_vs_rate_10_50_100_150"] = slo | {
        "non_increasing_2pp": {p: all(b <= a_ + 0.02 for a_, b in zip(x, x[1:])) for p, x in slo.items()}}
    # 4. consolidation: active nodes < 4 at light load, non-decreasing in rate and alpha
    act_rate = [run(r, 0.1, k)["active_nodes"] for r in (10.0, 50.0, 100.0, 150.0)]
    act_alpha = [run(10.0, al, k)["active_nodes"] for al in (0.1, 0.5, 0.9)]
    rep["active_nodes"] = {"vs_rate_alpha0.1": act_rate, "vs_alpha_rate10": act_alpha,
                           "light_load_below_4": act_rate[0] < 4.0,
                           "non_decreasing_0.25": all(b >= a_ - 0.25 for a_, b in zip(act_rate, act_rate[1:])) and
                           all(b >= a_ - 0.25 for a_, b in zip(act_alpha, act_alpha[1:]))}
    # 5. deprioritisation ablation ("w/o prioritize")
    on = run(100.0, 0.5, k)["slo_attainment"]
    off = run(100.0, 0.5, k, deprioritize=0)["slo_attainment"]
    rep["deprioritize_ablation_at_100"] = {"on": on, "off": off, "ratio": on / off if off > 0 else None}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
