# Round 2: compute-sanitizer over every kernel (tools/sanitize_run.py), then the full GPU suite,
# the default bench line and its launch list.
set -x
mkdir -p gpurun_out
rm -f gpurun_out/sanitize_summary.txt
timeout 300 python tools/sanitize_run.py > gpurun_out/sanitize_plain.txt 2>&1
bash tools/gpu_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:optimize_pipe --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1
