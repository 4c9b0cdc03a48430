# Round-2 deliverables in one GPU call: GPU tests, smoke (plain, serialised,
# under ncu), the default bench line, the reference arm, the Algorithm 2
# variant, the other BASELINE configs, the strong-scaling shard sizes, the ncu
# launch list of the bench and one ncu --set full capture of the MC kernel.
TAG=${1:-r02}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1; tail -2 $O/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke_ncu.log 2>&1; echo "ncu smoke rc=$?"
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; tail -1 $O/${TAG}_bench.err
timeout 900 python bench.py --impl reference > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
timeout 900 python bench.py --mem-cap 1024 --no-cpu > $O/${TAG}_bench_mem.json 2> $O/${TAG}_bench_mem.err
for c in sweep large paper mc-cb; do timeout 900 python bench.py --config $c >> $O/${TAG}_configs.jsonl 2>> $O/${TAG}_configs.err; done
for t in 32768 16384 8192; do timeout 600 python bench.py --traces $t --no-cpu --no-e2e >> $O/${TAG}_shards.jsonl 2>> $O/${TAG}_shards.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/${TAG}_launches_bench.json 2>&1; echo "ncu bench rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o $O/${TAG}_prof \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_prof.log 2>&1; echo "ncu full rc=$?"
ncu -i $O/${TAG}_prof.ncu-rep --page raw --csv > $O/${TAG}_prof_raw.csv 2>/dev/null
ncu -i $O/${TAG}_prof.ncu-rep --page source --csv --print-source cuda,sass > $O/${TAG}_prof_src.csv 2>/dev/null
ls -la $O | tail -30
