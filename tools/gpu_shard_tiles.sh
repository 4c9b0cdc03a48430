# Strong-scaling shard sizes on one GPU under different tile widths (lanes per
# trace; N = 4 nodes leave T - 4 idle lanes): does fewer traces per warp help
# the latency-bound small shards?
for t in 8192 16384; do for tl in 4 8 16; do
  LMX_TILE_LANES=$tl timeout 600 python bench.py --traces $t --no-cpu --no-e2e --steps 3 > gpurun_out/st_${t}_$tl.json 2> gpurun_out/st_${t}_$tl.err || tail -2 gpurun_out/st_${t}_$tl.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], 'kernel ms', round(d['kernel_ms_mean'],2), 'Gdec/s', round(d['value']/1e9,3), d['geometry'], d['parity'])" gpurun_out/st_${t}_$tl.json "traces=$t lanes=$tl"
done; done
