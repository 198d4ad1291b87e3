set -x
mkdir -p gpurun_out
grep -m1 -o -w -E 'fma|avx2' /proc/cpuinfo | head -2 > gpurun_out/host_flags.txt; lscpu | grep -m1 "Model name" >> gpurun_out/host_flags.txt; nproc >> gpurun_out/host_flags.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA -s > gpurun_out/pytest_gpu.txt 2>&1
