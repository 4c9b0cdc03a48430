# ncu --set full of the event-loop kernel for several library builds (bench
# config, 16,384 traces), exported as source pages.  Args: NAME=LIBSUFFIX
O=gpurun_out
for spec in "$@"; do
  name=${spec%%=*}; suf=${spec#*=}
  if [ "$suf" = "-" ]; then lib=$PWD/paper_2507_21276_b200/liblemix.so; else lib=$PWD/paper_2507_21276_b200/liblemix_$suf.so; fi
  LMX_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o $O/p_$name \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --traces ${TRACES:-16384} > $O/p_$name.log 2>&1
  ncu -i $O/p_$name.ncu-rep --page source --csv --print-source cuda,sass > $O/p_${name}_src.csv 2>/dev/null
  ncu -i $O/p_$name.ncu-rep --page raw --csv > $O/p_${name}_raw.csv 2>/dev/null
  rm -f $O/p_$name.ncu-rep
done
