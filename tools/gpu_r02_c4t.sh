# Config-4 stream timeline (full / pruned / probes-in-full-mode), the drop-in tests with the
# -fno-inline reference binaries, config 5 beside the queued config-2 line on the same box.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dropin_gpu.py -q -x > gpurun_out/pytest_dropin.txt 2>&1
timeout 900 python tools/c4_timeline.py > gpurun_out/c4_timeline.json 2> gpurun_out/c4_timeline.err
timeout 600 python bench.py --no-secondary --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 600 python bench.py --config c5 --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
