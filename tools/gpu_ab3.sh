# A/B of kernel variants on the bench workload: each arg is NAME=ENV1,ENV2 (ENV may set LMX_LIB=lib<suffix>)
set -u
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],1), 'Gdec/s', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],4), 'geom', d['geometry'], 'parity', d['parity'])" $1 $2; }
for spec in "$@"; do
  name=${spec%%=*}; envs=${spec#*=}
  envs=$(echo "$envs" | tr ',' ' ' | sed "s#LMX_LIB=lib#LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_#g; s#\(liblemix_[a-z0-9_]*\)#\1.so#g")
  [ "$envs" = "-" ] && envs=""
  if [ -n "${PARITY:-}" ]; then env $envs python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or paper or sweep" 2>&1 | tail -1; fi
  env $envs python bench.py --no-cpu --no-e2e --steps 3 --cpu-traces 64 > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err || tail -3 gpurun_out/ab_$name.err
  summ gpurun_out/ab_$name.json $name
done
