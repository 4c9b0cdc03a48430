bash tools/gpu_ab.sh base=- w8=w8 w2=w2 pf=pf
for c in sweep paper mc-cb large; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err || tail -5 gpurun_out/cfg_$c.err
  cut -c1-600 gpurun_out/cfg_$c.json
done
