# compute-sanitizer memcheck / racecheck / synccheck on small configs of every kernel path
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, workload
from paper_2507_21276_b200 import lemix
ef, eb = workload.profile(4, 2)
tr = workload.generate(workload.tiny_spec(rate=60.0, n_inf=150), 6, seed_base=3)
for kw in (dict(), dict(policy=lemix.LMX_RR), dict(policy=lemix.LMX_SEPARATE, sync_interval=3, sync_latency=0.2, sep_dynamic=1, dyn_rate=20.0, dyn_window=2.0),
           dict(mem_enable=1, mem_cap=300, mem_dt=0.0055, mem_tmax=0.055, mem_pen=1e-4), dict(qcap=3)):
    g = lemix.run(ef, eb, 4, 2, tr, lemix.Params(**kw), outputs=True)
    print(kw, "status", g.status)
ef8, eb8 = workload.profile(8, 8)
g = lemix.run(ef8, eb8, 8, 8, tr, lemix.Params(), outputs=True); print("8x8 status", g.status)
ef64, eb64 = workload.profile(64, 2)
g = lemix.run(ef64, eb64, 64, 2, tr, lemix.Params(), outputs=True); print("64x2 status", g.status)
# round 2: summary-only (LEAN) one-warp tiles and wide kernels (two-barrier decision),
# and the IEEE fallback of the division / sqrt fast paths (tiny tau)
for (N, S) in ((4, 2), (40, 8), (64, 2), (100, 4)):
    efn, ebn = workload.profile(N, S)
    for kw in (dict(), dict(tau=2.0 ** -1000), dict(qcap=3)):
        g = lemix.run(efn, ebn, N, S, tr, lemix.Params(**kw), outputs=False)
        print(N, S, "summary-only", kw, "status", g.status)
PY
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san.py 2>&1 | tail -4
done
