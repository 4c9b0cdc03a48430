# large-config A/B of library builds.  Args: NAME=LIBSUFFIX ("-" = liblemix.so)
O=gpurun_out
for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  LMX_LIB=$lib timeout 900 python bench.py --config large --steps 2 --warmup 1 > $O/lab_$name.json 2> $O/lab_$name.err || tail -3 $O/lab_$name.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'kernel', d['kernel_ms'], 'Mdec/s', round(d['value']/1e6,1), 'frac', round(d['roofline']['frac'],4))" $O/lab_$name.json $name
done
