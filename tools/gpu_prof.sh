# ncu --set full capture of the event-loop kernel (one launch) + source page export.
# Usage: tools/gpu_prof.sh TAG [TRACES] [LIBSUFFIX]
TAG=${1:-prof}; TR=${2:-16384}; SUF=${3:--}
O=gpurun_out
if [ "$SUF" = "-" ]; then export LMX_LIB=$PWD/paper_2507_21276_b200/liblemix.so; else export LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_$SUF.so; fi
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"(loop|lane)_kernel" -s 3 -c 1 -o $O/${TAG} \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --traces $TR > $O/${TAG}.log 2>&1
echo "ncu rc=$?"
ncu -i $O/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > $O/${TAG}_src.csv 2>/dev/null
ncu -i $O/${TAG}.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>/dev/null
ncu -i $O/${TAG}.ncu-rep --page details --csv > $O/${TAG}_details.csv 2>/dev/null
ncu -i $O/${TAG}.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ls -la $O/${TAG}*
