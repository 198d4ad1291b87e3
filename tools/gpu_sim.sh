set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sim_gpu.py -x -q > gpurun_out/pytest_sim.txt 2>&1
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
