"""Throughput of the large-cluster config (64 nodes x 8 stages, 296 traces of
200k requests + 200k training micro-batches) and of the sweep config, on the
product path (summary-only), for DESIGN.md.  Not the bench metric."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
import workload
from paper_2507_21276_b200 import lemix

def run(name, N, S, tr, lp, reps=2):
    ef, eb = workload.profile(N, S)
    ctx = lemix.Context(0)
    ctx.lmx_load_profile(N, S, ef, eb)
    ctx.lmx_load_traces(tr.offsets, tr.n_inf, tr.arrival, tr.lbk)
    ctx.lmx_set_params(lp)
    ctx.lmx_set_outputs(False)
    ks = []
    for _ in range(reps + 1):
        ctx.lmx_run(); assert ctx.lmx_sync() == 0, ctx.last_error()
        k_ms, r_ms, n = ctx.lmx_get_timing()
        ks.append(k_ms)
    g = ctx.lmx_get_geometry()
    ctx.close()
    k = min(ks[1:])
    print(json.dumps({"config": name, "decisions": int(tr.n_tasks), "traces": int(tr.n_traces), "kernel_ms": k,
                      "decisions_per_s": tr.n_tasks / (k / 1e3), "traces_per_s": tr.n_traces / (k / 1e3),
                      "geometry": g}), flush=True)

parts = [workload.generate(workload.large_spec(rate=r), 148, seed_base=7 + 148 * k) for k, r in enumerate((1600.0, 3200.0))]
run("large 64x8 (296 traces x 400k)", 64, 8, workload.concat(parts), lemix.Params(qcap=2048), reps=1)
for pol, nm in ((lemix.LMX_LEMIX, "lemix"), (lemix.LMX_RR, "rr"), (lemix.LMX_SEPARATE, "separate")):
    parts = [workload.generate(workload.sweep_spec(rate), 4096, seed_base=1 + 4096 * k) for k, rate in enumerate(workload.SWEEP_RATES)]
    run(f"sweep 4096x16 rates ({nm})", 4, 2, workload.concat(parts), lemix.Params(policy=pol))
