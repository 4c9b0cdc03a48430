"""Per-source-line aggregation of an ncu source page (cuda,sass CSV): top lines
by stall samples / executed instructions, and active threads per instruction."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ndec = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cur = None
hdr = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or len(r) < 8:
        continue
    if r[2] == '-':
        try:
            agg.append((cur, int(r[0]), r[1], float(r[4] or 0), float(r[7] or 0),
                        float(r[hdr.index("Thread Instructions Executed")] or 0)))
        except ValueError:
            pass
ti = sum(a[4] for a in agg)
ts = sum(a[3] for a in agg)
print(f"warp inst {ti:.4g}  per decision {ti / ndec:.1f}")
for a in sorted(agg, key=lambda a: -a[4])[:int(sys.argv[3]) if len(sys.argv) > 3 else 45]:
    print(f"{a[0][:12]:12} {a[1]:4} i{a[4] / ti * 100:5.1f}% s{a[3] / ts * 100:5.1f}% t{a[5] / max(1, a[4]):4.1f}"
          f" w/d {a[4] / ndec:5.1f} | {a[2].strip()[:85]}")
