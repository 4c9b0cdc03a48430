# per-trace time vs number of traces (persistent-grid tail effect)
for T in 18944 37888 56832 65536 75776; do
  python bench.py --no-cpu --no-e2e --steps 3 --cpu-traces 16 --traces $T > gpurun_out/tail_$T.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms', round(d['ms_per_step'],1), 'us/trace-round', round(d['ms_per_step']*1000/(int(sys.argv[2])/18944),1), 'Gdec/s', round(d['value']/1e9,3))" gpurun_out/tail_$T.json $T
done
