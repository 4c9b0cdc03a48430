"""The other BASELINE.json configurations on the product path, with the bench's
timing rules (python bench.py --config NAME delegates here; one JSON line).

  sweep  -- request-rate sweep: 4096 traces x 16 rates (10..160 tasks/s), 1,000
            tasks each, on identical traces under Separate, RR (NaiveMix) and
            LeMix; one step = the three policy runs; per-cell aggregates
  large  -- large cluster: 64 nodes x 8 stages, 296 traces (2 per SM) of 200k
            requests + 200k training micro-batches, heterogeneous lengths,
            400 -> 3200 tasks/s (half the traces at each end)
  paper  -- paper-scale: 10 seeds of the bursty 20k-request trace with 4,000
            continuous C = 4 training micro-batches, N = 4, S = 2
  mc-cb  -- the MC workload (65,536 traces, 10k + 10k tasks) with Algorithm 3
            continuous batching and decode steps (C = 8, T_w = 0.5 x the
            median request's inference latency; NEXT-2)

Each line carries decisions/s, traces/s, roofline (oracle event counters on a
sample x bench.OP_WEIGHTS for this N, S / the fp64 pipe peak), the sampled
bit-exact parity check and the clocks.  Inputs are device-resident and larger
than L2 (sweep: 0.8 GB; large: 1.4 GB; paper: 2.9 MB per seed, so L2 is
flushed between steps by a 256 MB write)."""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def op_weights(N, S):
    import bench
    D, Q, E = bench.DIV, bench.SQRT, bench.EXP
    w = {
        "decisions": 4, "stage_iters": 6, "scan_consumed": 4.5, "scan_break": 1, "offset_adds": 2,
        "alg1_calls": 1 + 4 + 3 + D + 1, "lc_exp": 3 + E + 1, "commits_train": 5 * S,
        "eq4_checks": 3 * N + 2 * S + 3, "version_scan": 1,
    }
    commit = 2 * S + (2 * D + Q + 6) + (3 + 2 * S + 1) / 2
    return w, commit


def ops_per_decision(counters, N, S):
    w, commit = op_weights(N, S)
    tot = sum(w[k] * counters[k] for k in w) + commit * counters["decisions"]
    return tot / max(1, counters["decisions"])


def build(name, seed=1):
    """(N, S, traces, [(label, Params)], eta_d, cells, n_cells, description)."""
    import workload
    from paper_2507_21276_b200 import lemix
    if name == "sweep":
        parts = [workload.generate(workload.sweep_spec(r), 4096, seed_base=seed + 4096 * k)
                 for k, r in enumerate(workload.SWEEP_RATES)]
        tr = workload.concat(parts)
        cells = np.repeat(np.arange(16, dtype=np.int32), 4096)
        runs = [("separate", lemix.Params(policy=lemix.LMX_SEPARATE)), ("rr", lemix.Params(policy=lemix.LMX_RR)),
                ("lemix", lemix.Params())]
        return (4, 2, tr, runs, None, cells, 16,
                "sweep: 4096 traces x 16 rates (10..160 tasks/s) x 1,000 tasks, N=4 x S=2, Llama-8B, "
                "Separate + RR + LeMix on identical traces, summary-only")
    if name == "large":
        half = 148
        parts = [workload.generate(workload.large_spec(rate=r), half, seed_base=seed + k * half)
                 for k, r in enumerate((1600.0, 3200.0))]
        tr = workload.concat(parts)
        return (64, 8, tr, [("lemix", lemix.Params(qcap=1024))], None, None, 1,
                "large: 296 traces (2 per SM) x (200k requests + 200k training), N=64 x S=8, Llama-8B "
                "(eta x 2/8), heterogeneous lengths (LogNormal 64, 1.5), 1600 / 3200 tasks/s, LeMix, summary-only")
    if name == "paper":
        tr = workload.generate(workload.paper_spec(), 10, seed_base=seed)
        return (4, 2, tr, [("lemix", lemix.Params())], None, None, 1,
                "paper: 10 seeds x (20k bursty CV=3 requests at 50 rps + 4,000 continuous C=4 training "
                "micro-batches), N=4 x S=2, Llama-8B, LeMix, summary-only")
    if name == "mc-cb":
        tr = workload.mc_traces(65536, seed_base=seed)
        lp = lemix.Params(cb_cmax=8, cb_tw=workload.batch_timeout(2), qcap=2048)
        return (4, 2, tr, [("lemix-cb", lp)], workload.decode_profile(4, 2), None, 1,
                "mc-cb: 65,536 traces x (10k requests + 10k training), N=4 x S=2, Llama-8B, LeMix with "
                "Algorithm 3 continuous batching (C=8, T_w=0.5 x the median request's forward = 1.8 ms) and decode steps (eta_D, LogNormal(200,1) "
                "output lengths), summary-only")
    raise SystemExit(f"unknown config {name}")


def run_config(name, args):
    import torch

    import bench
    import oracle
    import workload
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity_util import oracle_params
    from paper_2507_21276_b200 import lemix

    N, S, tr, runs, eta_d, cells, n_cells, desc = build(name, args.seed)
    ef, eb = workload.profile(N, S)
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    arr_d = torch.from_numpy(np.ascontiguousarray(tr.arrival)).to("cuda")
    lbk_d = torch.from_numpy(np.ascontiguousarray(tr.lbk).view(np.int32)).to("cuda")
    out_d = torch.from_numpy(np.ascontiguousarray(tr.out_len).view(np.int32)).to("cuda") if eta_d is not None else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if tr.n_tasks * 12 < (512 << 20) else None
    ctxs = []
    for label, lp in runs:
        ctx = lemix.Context(0, stream.cuda_stream)
        ctx.lmx_load_profile(N, S, ef, eb, eta_d)
        ctx.lmx_load_traces(tr.offsets, tr.n_inf, arr_d, lbk_d, mem=lemix.LMX_DEVICE, out_len=out_d)
        ctx.lmx_set_params(lp)
        ctx.lmx_set_cells(cells, n_cells)
        ctx.lmx_set_outputs(False)
        ctxs.append((label, lp, ctx))

    def step():
        ms = []
        for _, _, ctx in ctxs:
            ctx.lmx_run()
            st = ctx.lmx_sync()
            if st != lemix.LMX_OK:
                raise SystemExit(f"{name}: {ctx.last_error()}")
            ms.append(ctx.lmx_get_timing()[0])
        return ms

    for _ in range(args.warmup):
        step()
    sampler = bench.ClockSampler(0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern = []
    total = 0.0
    with sampler:
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1)
            torch.cuda.synchronize()
            ev0.record(stream)
            kern.append(step())
            ev1.record(stream)
            torch.cuda.synchronize()
            total += ev0.elapsed_time(ev1) / 1e3
    step_s = total / args.steps
    decisions = tr.n_tasks * len(runs)
    # parity on sampled traces + op counts for the roofline (oracle, as it stands)
    idx = np.unique(np.linspace(0, tr.n_traces - 1, min(tr.n_traces, 8 if N < 64 else 2)).astype(np.int64))
    if N >= 64:   # the oracle on a full 400k-task 64-node trace takes minutes: sample the first 20k tasks
        sub = workload.concat([workload.generate(workload.large_spec(rate=r, n_inf=10000), 1, seed_base=args.seed + k * 148)
                               for k, r in enumerate((1600.0, 3200.0))])
        idx = None
    else:
        sub = tr.subset(idx)
    parity = {"sampled_traces": int(sub.n_traces), "integers_exact": True, "fp64_bitwise": True}
    opd, counters_all = [], None
    for label, lp, ctx in ctxs:
        osum, _, counters, _ = oracle.run_batch(ef, eb, N, S, sub, oracle_params(lp), outputs=False, eta_d=eta_d)
        opd.append(ops_per_decision(counters, N, S))
        if idx is not None:
            g = ctx.lmx_get_summaries(tr.n_traces)[idx]
            for k in lemix.SUMMARY_INT:
                parity["integers_exact"] &= bool(np.array_equal(g[k], osum[k]))
            for k in lemix.SUMMARY_F64:
                parity["fp64_bitwise"] &= bool(np.array_equal(g[k].view(np.int64), osum[k].view(np.int64)))
    if idx is None:
        parity = {"sampled_traces": 0, "note": "large: parity of this shape is the -m gpu test test_large_sampled"}
    peaks, _ = bench.measured_peaks()
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    peak, peak_note = bench.fp64_peak(n_sm, mhz)
    k_s = [statistics.mean(k[r] for k in kern) / 1e3 for r in range(len(runs))]
    achieved = sum(o * tr.n_tasks for o in opd) / sum(k_s) / 1e12
    line = {"metric": bench.METRIC, "value": decisions / step_s, "unit": bench.UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "name": name, "traces": tr.n_traces, "tasks": tr.n_tasks,
                       "n_nodes": N, "n_stages": S, "policies": [r[0] for r in runs],
                       "l2": "inputs > L2" if flush is None else "L2 flushed (256 MB write) before each step"},
            "traces_per_s": tr.n_traces * len(runs) / step_s,
            "kernel_ms": {r[0]: round(k * 1e3, 3) for r, k in zip(runs, k_s)},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "peak_note": peak_note,
                         "ops_per_decision": {r[0]: round(o, 1) for r, o in zip(runs, opd)}},
            "parity": parity, "clocks": sampler.report()}
    print(json.dumps(line), flush=True)
    for _, _, ctx in ctxs:
        ctx.close()
