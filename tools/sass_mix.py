"""Dynamic instruction mix of one kernel from an ncu source page exported with
--print-source sass (per-SASS-instruction executed counts): totals by opcode,
and the hottest straight-line blocks.  Usage: sass_mix.py page.csv [decisions] [n]"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
ndec = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
iE, iT = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
ins = []
for r in rows[2:]:
    if len(r) < len(hdr) - 5:
        continue
    try:
        ins.append((int(r[0], 16), r[1].strip(), int(r[iE] or 0), int(r[iT] or 0), int(r[iS] or 0)))
    except ValueError:
        pass
tot = sum(x[2] for x in ins)
tst = sum(x[4] for x in ins)
print(f"warp instructions {tot:.4g} = {tot / ndec:.1f} per decision; {len(ins)} static")
ops = Counter()
for a, s, e, t, st in ins:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", s)
    op = m.group(2) if m else s.split()[0]
    ops[op] += e
for op, e in ops.most_common(30):
    print(f"{op:14} {e / tot * 100:5.1f}%  {e / ndec:6.1f}/dec")
print("--- blocks (offset, n instr, executions/decision, inst share, stall share)")
blocks = []
cur = None
for a, s, e, t, st in ins:
    if cur and e == cur[2]:
        cur[1] += 1
        cur[3] += e
        cur[4] += st
        cur[5].append(s)
    else:
        if cur:
            blocks.append(cur)
        cur = [a, 1, e, e, st, [s]]
blocks.append(cur)
base = ins[0][0]
for b in sorted(blocks, key=lambda b: -b[3])[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{b[0] - base:6x} n={b[1]:3} x{b[2] / ndec:8.4f}/dec  i{b[3] / tot * 100:5.1f}% s{b[4] / max(1, tst) * 100:5.1f}% | "
          + " ; ".join(x.split(" ")[0] if not x.startswith("@") else " ".join(x.split(" ")[:2]) for x in b[5][:8]))
