# strong-scaling shard sizes (one GPU) for library builds.  Args: NAME=LIBSUFFIX ("-" = liblemix.so)
for t in 8192 16384; do for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  LMX_LIB=$lib timeout 600 python bench.py --traces $t --no-cpu --no-e2e --steps 5 > gpurun_out/shab_${t}_$name.json 2> gpurun_out/shab_${t}_$name.err || tail -2 gpurun_out/shab_${t}_$name.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'kernel ms', round(d['kernel_ms_mean'],2), 'Gdec/s', round(d['value']/1e9,3), d['parity'])" gpurun_out/shab_${t}_$name.json "traces=$t $name"
done; done
