set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python tools/tune_search.py > gpurun_out/tune.txt 2>&1
