# ncu --set full of the wide kernel on the large config (one launch)
O=gpurun_out; TAG=${1:-large}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 1 -c 1 -o $O/p_$TAG \
  python bench.py --config large --steps 1 --warmup 1 > $O/p_$TAG.log 2>&1
ncu -i $O/p_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $O/p_${TAG}_src.csv 2>/dev/null
ncu -i $O/p_$TAG.ncu-rep --page raw --csv > $O/p_${TAG}_raw.csv 2>/dev/null
ncu -i $O/p_$TAG.ncu-rep --page details --csv > $O/p_${TAG}_details.csv 2>/dev/null
