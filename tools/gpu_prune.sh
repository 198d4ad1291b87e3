set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_sim_gpu.py tests/test_dropin_gpu.py -x -q > gpurun_out/pytest_prune.txt 2>&1; tail -2 gpurun_out/pytest_prune.txt
timeout 600 python tools/c4_phases.py 2>&1 | tail -1
for i in 1 2; do
timeout 900 python bench.py --config c4 --steps 5 --warmup 2 --no-cpu-baseline 2> gpurun_out/bench_c4.err | cut -c150-230
MISO_C4_FULL_STATIC=1 timeout 900 python bench.py --config c4 --steps 5 --warmup 2 --no-cpu-baseline 2> gpurun_out/bench_c4.err | cut -c150-230
done
