set -x
mkdir -p gpurun_out
timeout 1500 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
