for v in tile lane; do
  if [ $v = tile ]; then export LMX_KERNEL=tile; else unset LMX_KERNEL; export LMX_LIB=$PWD/paper_2507_21276_b200/liblemix_mb2.so; fi
  ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o gpurun_out/p2_$v python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p2_$v.log 2>&1
done
