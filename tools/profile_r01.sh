set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r01_launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:event_loop -s 3 -c 1 -o gpurun_out/r01_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r01_prof_bench.log 2>&1
ls -la gpurun_out
