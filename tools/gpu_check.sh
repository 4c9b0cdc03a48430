# Quick GPU check: full GPU tests, smoke under ncu (serialised streams) and
# with one hardware queue, then one bench line.  Usage: tools/gpu_check.sh TAG
TAG=${1:-chk}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.txt 2>&1; tail -3 $O/${TAG}_pytest_gpu.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_smoke_launches.csv \
    python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke_ncu.log 2>&1; echo "smoke under ncu rc=$?"; tail -1 $O/${TAG}_smoke_ncu.log
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; tail -2 $O/${TAG}_bench.err; cut -c1-400 $O/${TAG}_bench.json
