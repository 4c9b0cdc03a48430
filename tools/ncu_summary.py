#!/usr/bin/env python
"""Summarise an ncu report of the event-loop kernel into profiles/.

    python tools/ncu_summary.py <report.ncu-rep> <out-prefix> [--traces T --tasks M]

Writes <out-prefix>.txt (speed-of-light, occupancy, stall reasons, pipe
utilisation, DRAM bytes, top source lines) and, with --traces/--tasks,
profiles/traffic.json (DRAM bytes per launch for bench.py's roofline).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess

DETAILS = ("Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Achieved Active Warps Per SM",
           "Theoretical Occupancy", "Executed Ipc Active", "Issue Slots Busy", "Avg. Active Threads Per Warp",
           "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate",
           "DRAM Throughput", "Memory Throughput", "Executed Instructions", "Grid Size", "Block Size",
           "Dynamic Shared Memory Per Block")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum")


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traces", type=int, default=0)
    ap.add_argument("--tasks", type=int, default=0)
    a = ap.parse_args()
    lines = [f"# ncu summary of {os.path.basename(a.report)}", ""]
    det = list(csv.reader(io.StringIO(ncu("-i", a.report, "--page", "details", "--csv"))))
    hdr = det[0]
    kname = None
    for r in det[1:]:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in DETAILS:
            lines.append(f"{d['Metric Name']:38s} {d['Metric Value']:>18s} {d.get('Metric Unit', '')}")
    lines.insert(1, f"kernel: {kname}")
    raw = list(csv.reader(io.StringIO(ncu("-i", a.report, "--page", "raw", "--csv"))))
    rd = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
    units = dict(zip(raw[0], raw[1])) if len(raw) > 2 else {}
    lines += ["", "## raw counters"]
    for k in RAW:
        lines.append(f"{k:70s} {rd.get(k)} {units.get(k, '')}")
    stalls = {k: float(v) for k, v in rd.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    lines += ["", "## stall reasons (warps stalled per issued instruction)"]
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        lines.append(f"{v:8.3f}  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
    # top source lines
    src = list(csv.reader(io.StringIO(ncu("-i", a.report, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur = None
    h = None
    agg = {}
    for r in src:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if h is None or len(r) < 5 or r[2] != "-":
            continue
        try:
            ln = int(r[0])
            inst = float(r[h.index("Instructions Executed")])
            samp = float(r[h.index("Warp Stall Sampling (All Samples)")])
            thr = float(r[h.index("Thread Instructions Executed")])
        except (ValueError, IndexError):
            continue
        agg[(cur, ln)] = (inst, samp, thr, r[1].strip()[:90])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    lines += ["", "## top source lines by stall samples (inst% / samples% / avg active threads)"]
    for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        lines.append(f"{f}:{ln:<5d} {100 * v[0] / ti:5.1f}% {100 * v[1] / ts:5.1f}% thr={v[2] / max(v[0], 1):5.1f}  {v[3]}")
    with open(a.out + ".txt", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))
    if a.traces and a.tasks:
        def to_bytes(k):
            v = float(rd.get(k, 0) or 0)
            u = units.get(k, "byte").lower()
            return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)
        tb = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
        out = {"traces": a.traces, "tasks_per_trace": a.tasks, "dram_bytes_per_launch": tb,
               "source": os.path.basename(a.report), "kernel": kname}
        with open(os.path.join(os.path.dirname(a.out) or ".", "traffic.json"), "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
