# sweep-config A/B of library builds.  Args: NAME=LIBSUFFIX ("-" = liblemix.so)
O=gpurun_out
for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  LMX_LIB=$lib timeout 900 python bench.py --config sweep --steps 5 --warmup 3 > $O/sab_$name.json 2> $O/sab_$name.err || tail -3 $O/sab_$name.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],2), 'kernel', d.get('kernel_ms'), 'Gdec/s', round(d['value']/1e9,3), 'parity', d.get('parity'))" $O/sab_$name.json $name
done
