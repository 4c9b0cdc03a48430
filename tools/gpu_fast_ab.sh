# Fast-kernel iteration: full GPU tests (fast kernel is the default where it
# applies), then bench A/B: fast vs LMX_KERNEL=generic.
O=gpurun_out; TAG=${1:-fa}
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.txt 2>&1; tail -3 $O/${TAG}_pytest.txt
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],1), 'kernel', round(d['kernel_ms_mean'],1), 'Gdec/s', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],4), 'geom', d['geometry'], 'parity', d['parity'])" $1 $2; }
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > $O/${TAG}_fast.json 2> $O/${TAG}_fast.err || tail -3 $O/${TAG}_fast.err; summ $O/${TAG}_fast.json fast
LMX_KERNEL=generic timeout 600 python bench.py --no-cpu --no-e2e --steps 3 > $O/${TAG}_gen.json 2> $O/${TAG}_gen.err || tail -3 $O/${TAG}_gen.err; summ $O/${TAG}_gen.json generic
if [ "${NCU:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o $O/${TAG}_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_prof.log 2>&1
ncu -i $O/${TAG}_prof.ncu-rep --page source --csv --print-source cuda,sass > $O/${TAG}_src.csv 2>/dev/null
ncu -i $O/${TAG}_prof.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
fi
