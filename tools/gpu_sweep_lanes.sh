# sweep config under different lanes-per-trace (LMX_TILE_LANES): per-policy kernel times
for tl in 4 2 1; do
  LMX_TILE_LANES=$tl timeout 900 python bench.py --config sweep --steps 5 --warmup 3 > gpurun_out/sl_$tl.json 2> gpurun_out/sl_$tl.err || tail -3 gpurun_out/sl_$tl.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('lanes', sys.argv[2], 'ms/step', round(d['ms_per_step'],2), 'kernel', d.get('kernel_ms'), 'parity', d.get('parity'))" gpurun_out/sl_$tl.json $tl
done
