set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_prune.txt 2>&1; tail -2 gpurun_out/pytest_prune.txt
for i in 1 2; do timeout 600 python tools/c4_phases.py 2>&1 | tail -1; done
timeout 900 python bench.py --config c4 --steps 5 --warmup 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; cut -c1-400 gpurun_out/bench_c4.json
