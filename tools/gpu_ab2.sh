set -u
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
summ() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'ms/step', round(d['ms_per_step'],1), 'Gdec/s', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],4), 'geom', d['geometry'], 'parity', d['parity'])" $1 $2; }
for v in "$@"; do
  case $v in
    default) env="" ;;
    lane) env="LMX_KERNEL=lane" ;;
    T2) env="LMX_TILE_LANES=2" ;;
    T1) env="LMX_TILE_LANES=1" ;;
    lanemb2) env="LMX_KERNEL=lane LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_mb2.so" ;;
    T2t3) env="LMX_TILE_LANES=2 LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_t3.so" ;;
    *) env="LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_$v.so" ;;
  esac
  env $env python bench.py --no-cpu --no-e2e --steps 3 --cpu-traces 64 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err || tail -3 gpurun_out/ab_$v.err
  summ gpurun_out/ab_$v.json $v
done
