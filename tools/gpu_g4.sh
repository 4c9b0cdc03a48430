timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest.txt 2>&1; tail -15 gpurun_out/g4_pytest.txt
bash tools/gpu_ab.sh base=-
