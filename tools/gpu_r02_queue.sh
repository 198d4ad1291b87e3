# Queued search launches (miso_b200_optimize_batches): tests, the default bench line without
# secondary configs, its launch list, and one ncu --set full capture of a 32-step launch.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search_gpu.py -q -x > gpurun_out/pytest_search.txt 2>&1
timeout 600 python bench.py --no-secondary > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:optimize_pipe --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 64 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch_q.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:optimize_pipe -s 1 -c 1 -o gpurun_out/search_queue -f python tools/search_queue_once.py 32 > gpurun_out/ncu_queue.log 2>&1
