# one iteration: parity tests, bench, ncu capture of the event-loop kernel
TAG=${1:-iter}
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
python bench.py --no-cpu > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err
python - <<'PY' gpurun_out/${TAG}_bench.json
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","kernel_ms_mean","traces_per_s")}, d["roofline"]["frac"] if d.get("roofline") else None, d.get("e2e",{}).get("value"), d.get("geometry"), d.get("parity"))
PY
if [ "${NCU:-1}" = "1" ]; then
ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --traces ${NCU_TRACES:-16384} > gpurun_out/${TAG}_prof.log 2>&1
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Active Warps Per SM|Executed Ipc Active|Avg. Active Threads Per Warp|L1/TEX Hit Rate|L2 Hit Rate|DRAM Throughput|Issue Slots Busy|Executed Instructions|Eligible Warps Per Scheduler)"' | awk -F'","' '{print $(NF-2)" = "$NF}'
fi
