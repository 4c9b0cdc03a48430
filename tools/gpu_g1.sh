PARITY=1 bash tools/gpu_ab.sh base=- m5=m5
for t in 8192 16384 32768; do TRACES=$t bash tools/gpu_ab.sh base_$t=-; done
