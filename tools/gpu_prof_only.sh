# one ncu --set full capture of the event-loop kernel at the bench config (16384 traces) + SASS-level source page
TAG=${1:-prof}
ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 3 -c 1 -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --traces ${NCU_TRACES:-16384} > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Active Warps Per SM|Executed Ipc Active|Avg. Active Threads Per Warp|Issue Slots Busy|Executed Instructions|Eligible Warps Per Scheduler|Warp Cycles Per Issued Instruction|DRAM Throughput)"' | awk -F'","' '{print $(NF-2)" = "$NF}'
