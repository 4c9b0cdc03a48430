# A/B of library builds on the bench workload.  Args: NAME=LIBSUFFIX ("-" = liblemix.so)
# Optional env: TRACES (default 65536), PARITY=1 runs the parity tests per build first.
set -u
O=gpurun_out
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],1), 'kernel', round(d['kernel_ms_mean'],1), 'Gdec/s', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],4) if d.get('roofline') else None, 'geom', d['geometry'], 'parity', d['parity'], 'clk', d['clocks'].get('sm_mhz'))" $1 $2; }
for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  if [ -n "${PARITY:-}" ]; then LMX_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepwise.py -x -q 2>&1 | tail -1; fi
  LMX_LIB=$lib timeout 900 python bench.py --no-cpu --no-e2e --steps 3 --cpu-traces 64 --traces ${TRACES:-65536} > $O/ab_$name.json 2> $O/ab_$name.err || tail -3 $O/ab_$name.err
  summ $O/ab_$name.json $name
done
