# round deliverables: tests, full bench line, launch list, ncu full capture
TAG=${1:-r01}
python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; cat gpurun_out/${TAG}_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/${TAG}_prof.log 2>&1
ls -la gpurun_out
