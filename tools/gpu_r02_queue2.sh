# Queued search launches with descriptors prepared before the timed region; c4 with the pruned
# chosen-only static search (A/B against the default full search on the same box).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py -q -x -k batches > gpurun_out/pytest_search.txt 2>&1
timeout 600 python bench.py --no-secondary > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 600 python bench.py --no-secondary --steps 64 > gpurun_out/bench_q64.json 2> gpurun_out/bench_q64.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/c4_full.json 2> gpurun_out/c4_full.err
MISO_C4_PRUNED_STATIC=1 timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/c4_pruned.json 2> gpurun_out/c4_pruned.err
