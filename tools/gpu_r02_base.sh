# Round-2 baseline in one GPU call: GPU tests, smoke (plain, under ncu, and
# serialised with CUDA_DEVICE_MAX_CONNECTIONS=1 -- the host-input deadlock
# check), the default bench line, the ncu launch list of the bench (with the
# e2e leg) and one ncu --set full capture of the event-loop kernel.
TAG=${1:-r02}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.txt 2>&1; tail -2 $O/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1; echo "serialised smoke rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke_ncu.log 2>&1; echo "ncu smoke rc=$?"
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; tail -1 $O/${TAG}_bench.err; cat $O/${TAG}_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/${TAG}_launches_bench.json 2>&1; echo "ncu bench rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o $O/${TAG}_prof \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_prof.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/${TAG}_prof.ncu-rep --page raw --csv > $O/${TAG}_prof_raw.csv 2>/dev/null
ncu -i $O/${TAG}_prof.ncu-rep --page details --csv > $O/${TAG}_prof_details.csv 2>/dev/null
ncu -i $O/${TAG}_prof.ncu-rep --page source --csv --print-source sass > $O/${TAG}_prof_sass.csv 2>/dev/null
ls -la $O | tail -30
