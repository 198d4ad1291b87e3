# Scalar optimize_partition through the resident server: search GPU tests, drop-in tests, c1 line.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py tests/test_dropin_gpu.py tests/test_predict_gpu.py -q -x > gpurun_out/pytest_c1.txt 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
