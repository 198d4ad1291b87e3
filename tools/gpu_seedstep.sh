set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; head -c 400 gpurun_out/bench_c3.json
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; head -c 400 gpurun_out/bench_c1.json
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; head -c 300 gpurun_out/bench_c4.json
