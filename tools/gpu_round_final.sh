# Round deliverables in one GPU call: full GPU tests + smoke, bench lines
# (default, Algorithm 2 variant, reference arm), the ncu launch list of the
# bench command and one ncu --set full capture of the event-loop kernel.
TAG=${1:-r01}
O=gpurun_out
python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.txt 2>&1; tail -2 $O/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; tail -1 $O/${TAG}_bench.err
python bench.py --mem-cap 1024 > $O/${TAG}_bench_mem.json 2> $O/${TAG}_bench_mem.err; tail -1 $O/${TAG}_bench_mem.err
python bench.py --impl reference > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o $O/${TAG}_prof \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_prof.log 2>&1
ls -la $O | tail -20
