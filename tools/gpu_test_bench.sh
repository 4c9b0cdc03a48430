set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
