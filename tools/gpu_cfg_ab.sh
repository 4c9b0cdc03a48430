# A/B of library builds on bench configs.  Usage: CFG="mc-cb" bash tools/gpu_cfg_ab.sh NAME=LIBSUFFIX ...
O=gpurun_out
for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  LMX_LIB=$lib timeout 900 python bench.py $ARGS --steps 3 --warmup 3 --no-cpu --no-e2e > $O/cab_$name.json 2> $O/cab_$name.err || tail -3 $O/cab_$name.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], sys.argv[3], 'ms/step', round(d['ms_per_step'],2), 'Gdec/s', round(d['value']/1e9,3), 'parity', d.get('parity'))" $O/cab_$name.json $name "$ARGS"
done
