# Round-2 validation of the current tree: sanitizers over every kernel, the full GPU suite,
# smoke, the default bench line (all secondary configs), the reference arm, the 2-rank
# self-spawned bench and the launch list.
set -x
mkdir -p gpurun_out
rm -f gpurun_out/sanitize_summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python tools/sanitize_run.py > gpurun_out/sanitize_plain.txt 2>&1
bash tools/gpu_sanitize.sh
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --gpus 2 --no-secondary > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:optimize_pipe --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1
