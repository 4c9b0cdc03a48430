timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stepwise.py tests/test_golden.py -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_ab.sh lane=-
TRACES=8192 bash tools/gpu_ab.sh lane_8192=-
