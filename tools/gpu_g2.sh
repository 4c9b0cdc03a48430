timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g2_pytest.txt 2>&1; tail -3 gpurun_out/g2_pytest.txt
bash tools/gpu_ab.sh lane=-
LMX_KERNEL=tile bash tools/gpu_ab.sh tile=-
for t in 8192 16384 32768; do TRACES=$t bash tools/gpu_ab.sh lane_$t=-; done
