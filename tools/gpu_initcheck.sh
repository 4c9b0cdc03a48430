for cfg in "policy=lemix.LMX_RR" "policy=lemix.LMX_SEPARATE,sync_interval=3,sync_latency=0.2,sep_dynamic=1,dyn_rate=20.0,dyn_window=2.0" "mem_enable=1,mem_cap=300,mem_dt=0.0055,mem_tmax=0.055,mem_pen=1e-4" "qcap=3"; do
echo "== $cfg"
timeout 300 compute-sanitizer --tool initcheck --print-limit 3 python -c "
import sys; sys.path.insert(0, '.')
import workload
from paper_2507_21276_b200 import lemix
ef, eb = workload.profile(4, 2)
tr = workload.generate(workload.tiny_spec(rate=60.0, n_inf=150), 6, seed_base=3)
print(lemix.run(ef, eb, 4, 2, tr, lemix.Params($cfg), outputs=True).status)" 2>&1 | grep -E "ERROR SUMMARY|Uninitialized|at .*0x|by thread|Host API|^[0-9]" | head -8
done
